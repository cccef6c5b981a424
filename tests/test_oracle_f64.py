"""Pins of the oracle's fp64 build (liboracle_f64.so, or_val = double).

The paper's streams carry "single or double precision floating point values"
(§5.1).  The same simulator source is compiled with double values;
these tests pin that build against exact arithmetic (dyadic values whose
partial sums are all representable in fp64 but not in fp32), the canonical
summation tree (R-8) through an order-sensitive example, the dense-switch
formula with isize = 8, the wire sizes, and numpy's max/min.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle

F64 = np.float64


def test_builds_have_their_value_sizes():
    assert oracle.lib(False).or_val_bytes() == 4
    assert oracle.lib(True).or_val_bytes() == 8


def test_merge_keeps_bits_fp32_would_drop():
    # 1 + 2^-30 and 2^-30 are exact in fp64; their sum 1 + 2^-29 too -- fp32 rounds both to 1
    a = 1.0 + 2.0 ** -30
    i, v = oracle.merge_sum([3], [a], [3, 7], [2.0 ** -30, 5.0], dtype=F64)
    assert list(i) == [3, 7]
    assert v.dtype == F64
    assert v[0] == 1.0 + 2.0 ** -29 and v[1] == 5.0
    i32, v32 = oracle.merge_sum([3], [a], [3], [2.0 ** -30])
    assert v32[0] == np.float32(1.0)


def _dyadic_streams(P, N, k, seed):
    """Sorted unique supports; values m * 2^-40 with |m| < 2^40: every partial
    sum over <= 16 ranks is an integer multiple of 2^-40 below 2^45 * 2^-40,
    so fp64 adds it exactly in any order (fp32 would not)."""
    g = np.random.default_rng(seed)
    out = []
    for _ in range(P):
        idx = np.sort(g.choice(N, size=k, replace=False)).astype(np.uint32)
        m = g.integers(-(1 << 40), 1 << 40, size=k)
        out.append((idx, (m.astype(np.float64) * 2.0 ** -40)))
    return out


def _exact(N, streams):
    acc, mask = {}, np.zeros(N, bool)
    for idx, val in streams:
        for x, v in zip(idx, val):
            acc[int(x)] = acc.get(int(x), Fraction(0)) + Fraction(float(v))
            mask[x] = True
    return acc, mask


def _check(res, N, acc, mask):
    d, i, v = res
    if d:
        for x in range(N):
            assert Fraction(float(v[x])) == acc.get(x, Fraction(0))
    else:
        assert list(i) == sorted(acc)
        for x, y in zip(i, v):
            assert Fraction(float(y)) == acc[int(x)]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 7, 8])
@pytest.mark.parametrize("k", [0, 5, 40, 150])
def test_collectives_exact_on_dyadic_values(P, k):
    N = 300
    streams = _dyadic_streams(P, N, min(k, N), seed=10 * P + k)
    acc, mask = _exact(N, streams)
    for algo in (oracle.ALGO_SSAR_SPLIT, oracle.ALGO_DSAR_SPLIT, oracle.ALGO_AUTO):
        res, _, _ = oracle.split_allgather(N, streams, algo=algo, dtype=F64)
        assert all(r[2].dtype == F64 for r in res)
        for r in res:
            _check(r, N, acc, mask)
    res, _ = oracle.ssar_recursive_double(N, streams, dtype=F64)
    for r in res:
        _check(r, N, acc, mask)


def test_fp32_build_is_not_exact_on_the_same_values():
    # guards the test above: the dyadic values do lose bits in fp32
    N = 300
    streams = _dyadic_streams(4, N, 40, seed=3)
    acc, _ = _exact(N, streams)
    res, _, _ = oracle.split_allgather(N, [(i, v.astype(np.float32)) for i, v in streams], algo=oracle.ALGO_SSAR_SPLIT)
    d, i, v = res[0]
    assert any(Fraction(float(y)) != acc[int(x)] for x, y in zip(i, v))


def test_canonical_tree_order_in_fp64():
    # P = 4, one index, values (1, 0, 2^-53, 2^-53): tree ((r0 + r1) + (r2 + r3))
    # (R-8) = 1 + 2^-52, while the left-to-right sum ((r0 + r1) + r2) + r3 = 1
    # (ties to even drop 2^-53 twice)
    u = 2.0 ** -53
    vals = [1.0, 0.0, u, u]
    streams = [(np.array([2], np.uint32), np.array([x])) for x in vals]
    assert ((1.0 + 0.0) + u) + u == 1.0 and (1.0 + 0.0) + (u + u) == 1.0 + 2 * u
    res, _, _ = oracle.split_allgather(8, streams, algo=oracle.ALGO_SSAR_SPLIT, dtype=F64)
    assert res[0][2][0] == 1.0 + 2 * u
    # recursive doubling at P = 4 associates the same way (stage 1: pairs, stage 2: halves)
    res, _ = oracle.ssar_recursive_double(8, streams, dtype=F64)
    for d, i, v in res:
        assert v[0] == 1.0 + 2 * u


def test_switch_threshold_with_double_values():
    # delta = floor(N * isize / (c + isize)): isize 8, c 4 -> 2N/3
    assert oracle.switch_threshold(12, isize=8) == 8
    assert oracle.switch_threshold(12) == 6
    N = 12
    # K = 7 pairs: sparse in fp64 (7 <= 8), dense in fp32 (7 > 6)
    s = [(np.array([0, 2, 4, 6], np.uint32), np.ones(4)), (np.array([1, 3, 5], np.uint32), np.ones(3))]
    r64, _, _ = oracle.split_allgather(N, s, algo=oracle.ALGO_SSAR_SPLIT, dtype=F64)
    r32, _, _ = oracle.split_allgather(N, s, algo=oracle.ALGO_SSAR_SPLIT)
    assert r64[0][0] is False and len(r64[0][1]) == 7
    assert r32[0][0] is True
    # K = 9 > 8: dense in fp64 too, zeros off the union
    s2 = s + [(np.array([7, 8], np.uint32), np.ones(2))]
    r64, _, _ = oracle.split_allgather(N, s2, algo=oracle.ALGO_SSAR_SPLIT, dtype=F64)
    assert r64[0][0] is True
    assert list(r64[0][2]) == [1.0] * 9 + [0.0] * 3


def test_wire_bytes_count_twelve_per_pair():
    N = 64
    s = [(np.array([1, 40], np.uint32), np.ones(2)), (np.array([2], np.uint32), np.ones(1))]
    _, st, _ = oracle.split_allgather(N, s, algo=oracle.ALGO_SSAR_SPLIT, dtype=F64)
    # rank 0 sends its index 40 (partition 1) = 1 pair, then its partition result {1, 2} = 2 pairs
    assert st[0]["bytes_sent"] == 12 * (1 + 2)
    _, st, _ = oracle.split_allgather(N, s, algo=oracle.ALGO_DSAR_SPLIT, dtype=F64)
    # DSAR: the dense partition of 32 words, 8 bytes each
    assert st[0]["bytes_sent"] == 12 * 1 + 8 * 32
    _, st = oracle.sparse_allgather(N, [(np.array([1], np.uint32), np.ones(1)),
                                        (np.array([40], np.uint32), np.ones(1))], dtype=F64)
    assert st[0]["bytes_sent"] == 12 and st[0]["bytes_recv"] == 12


def test_qsgd_is_not_defined_on_the_fp64_build():
    s = [(np.array([1], np.uint32), np.ones(1)), (np.array([2], np.uint32), np.ones(1))]
    with pytest.raises(ValueError):
        oracle.split_allgather(64, s, algo=oracle.ALGO_DSAR_SPLIT, quant_bits=4, dtype=F64)


@pytest.mark.parametrize("op", [oracle.OP_MAX, oracle.OP_MIN])
def test_max_min_match_numpy_in_fp64(op):
    N, P = 200, 5
    streams = _dyadic_streams(P, N, 60, seed=op)
    fill = -np.inf if op == oracle.OP_MAX else np.inf
    M = np.full((P, N), fill)
    for r, (i, v) in enumerate(streams):
        M[r, i] = v
    ref = M.max(axis=0) if op == oracle.OP_MAX else M.min(axis=0)
    mask, bf = oracle.brute_force_op(N, streams, op, dtype=F64)
    np.testing.assert_array_equal(bf, ref)
    with oracle.op_scope(op):
        res, _, _ = oracle.split_allgather(N, streams, algo=oracle.ALGO_DSAR_SPLIT, dtype=F64)
    np.testing.assert_array_equal(res[0][2], ref)


def test_explicit_zero_from_cancellation_is_kept():
    # an index in the union stays in the result even if its sum is 0
    x = 1.0 + 2.0 ** -40
    s = [(np.array([5], np.uint32), np.array([x])), (np.array([5, 9], np.uint32), np.array([-x, 2.0]))]
    res, _, _ = oracle.split_allgather(32, s, algo=oracle.ALGO_SSAR_SPLIT, dtype=F64)
    assert list(res[0][1]) == [5, 9] and list(res[0][2]) == [0.0, 2.0]
