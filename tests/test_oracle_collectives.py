"""Pins for the oracle's collective simulators (§5.3).

The simulators are checked against: the cited worked examples; the exact
volume closed forms of recursive doubling and DSAR;
the plain definition (numpy dense scatter-add) on many random small cases;
the paper's invariants (sorted unique indices, max k_i <= K <= min(N, sum k),
replicas identical); and the App. B expected result size."""
import json
import os

import numpy as np
import pytest

from paper_1802_08021_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _streams(lst):
    out = []
    for s in lst:
        a = np.array(s, dtype=np.float64).reshape(-1, 2)
        out.append((a[:, 0].astype(np.uint32), a[:, 1].astype(np.float32)))
    return out


def _dense_ref(N, streams):
    acc = np.zeros(N, np.float64)
    absacc = np.zeros(N, np.float64)
    mask = np.zeros(N, bool)
    for idx, val in streams:
        np.add.at(acc, idx.astype(np.int64), val.astype(np.float64))
        np.add.at(absacc, idx.astype(np.int64), np.abs(val.astype(np.float64)))
        mask[idx] = True
    return mask, acc, absacc


def _check_against_definition(N, streams, results, exact, delta):
    """Every replica equals the dense definition; sparse results obey the
    stream invariants.  Tolerance for float inputs: the
    summation order differs from a left fold, |g-o| <= 1e-5|o| + P*2^-24*S."""
    P = len(streams)
    mask, acc, absacc = _dense_ref(N, streams)
    K = int(mask.sum())
    ks = [len(s[0]) for s in streams]
    assert max(ks + [0]) <= K <= min(N, sum(ks))
    for r, (d, i, v) in enumerate(results):
        if d:
            vec = v.astype(np.float64)
            assert vec.shape == (N,)
            assert np.all(vec[~mask] == 0)
            got = vec[mask]
        else:
            assert len(i) == K, "K must equal |union H_i| exactly (P:459-461)"
            assert len(i) <= delta, "sparse implies nnz <= delta (S:89)"
            np.testing.assert_array_equal(i, np.nonzero(mask)[0])
            got = v.astype(np.float64)
        want = acc[mask]
        if exact:
            np.testing.assert_array_equal(got, want)
        else:
            tol = 1e-5 * np.abs(want) + P * 2.0 ** -24 * absacc[mask]
            assert np.all(np.abs(got - want) <= tol)
        d0, i0, v0 = results[0]
        assert d == d0
        if not d:
            np.testing.assert_array_equal(i, i0)
        np.testing.assert_array_equal(v, v0)   # replicas identical; -0 == +0


def test_rd_example(orc):
    ex = _load("collectives_examples.json")["rd_p2"]
    res, st = orc.ssar_recursive_double(ex["N"], _streams(ex["streams"]))
    for d, i, v in res:
        assert not d
        np.testing.assert_array_equal(i, [0])
        np.testing.assert_array_equal(v, [3.0])


def test_split_example(orc):
    ex = _load("collectives_examples.json")["split_p2"]
    res, st, dsar = orc.split_allgather(ex["N"], _streams(ex["streams"]), algo=orc.ALGO_SSAR_SPLIT)
    assert not dsar
    for d, i, v in res:
        np.testing.assert_array_equal(i, [0, 1])
        np.testing.assert_array_equal(v, [1.0, 2.0])
    # phase 1: P-1 messages per rank; phase 2: P-1 more
    assert all(s["msgs_sent"] == 2 * ex["phase1_msgs_per_rank"] for s in st)


def test_dsar_example(orc):
    ex = _load("collectives_examples.json")["dsar_p2"]
    res, st, dsar = orc.split_allgather(ex["N"], _streams(ex["streams"]), algo=orc.ALGO_DSAR_SPLIT)
    assert dsar
    for d, i, v in res:
        assert d
        np.testing.assert_array_equal(v, ex["dense_out"])


def test_rd_volume_extremes(orc):
    """Exact pair volumes per rank: log2(P)*k for identical supports and
    k(P-1) for disjoint ones."""
    ex = _load("collectives_examples.json")["rd_volume"]
    P, k, N = ex["P"], ex["k"], 1024
    _, st = orc.ssar_recursive_double(N, synth.disjoint_streams(P, N, k, seed=2))
    assert all(s["pairs_sent"] == ex["disjoint_pairs_per_rank"] for s in st)
    _, st = orc.ssar_recursive_double(N, synth.identical_streams(P, N, k, seed=2))
    assert all(s["pairs_sent"] == ex["identical_pairs_per_rank"] for s in st)
    # general P: the closed forms
    for P in [2, 4, 16]:
        _, st = orc.ssar_recursive_double(4096, synth.disjoint_streams(P, 4096, 7, seed=P))
        assert all(s["pairs_sent"] == 7 * (P - 1) for s in st)
        _, st = orc.ssar_recursive_double(4096, synth.identical_streams(P, 4096, 7, seed=P))
        assert all(s["pairs_sent"] == 7 * int(np.log2(P)) for s in st)


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("P", [2, 4, 8])
def test_rd_matches_definition(orc, seed, P):
    rng = np.random.default_rng(100 * P + seed)
    N = int(rng.choice([64, 500, 4096]))
    d = float(rng.choice([0.001, 0.01, 0.1, 0.3]))
    k = max(1, int(d * N))
    kind = "int" if seed % 2 == 0 else "normal"
    streams = synth.uniform_streams(P, N, k, seed=seed, kind=kind)
    delta = orc.switch_threshold(N)
    res, st = orc.ssar_recursive_double(N, streams)
    _check_against_definition(N, streams, res, kind == "int", delta)
    # stage sizes are non-decreasing and the switch fires only above delta
    for s in st:
        nnz = [s["stage_nnz"][t] for t in range(int(np.log2(P)))]
        assert nnz == sorted(nnz)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("P", [1, 2, 3, 4, 6, 8, 16])
@pytest.mark.parametrize("algo", [2, 3, 0])
def test_split_matches_definition(orc, seed, P, algo):
    rng = np.random.default_rng(1000 * P + 10 * algo + seed)
    N = int(rng.choice([64, 4096, 65536]))
    if N < P:
        N = 64
    d = float(rng.choice([0.001, 0.01, 0.1]))
    k = max(1, int(d * N))
    kind = "int" if seed % 2 == 0 else "normal"
    streams = synth.uniform_streams(P, N, k, seed=seed, kind=kind)
    delta = orc.switch_threshold(N)
    res, st, dsar = orc.split_allgather(N, streams, algo=algo)
    _check_against_definition(N, streams, res, kind == "int", delta)
    if algo == 0:
        assert dsar == (P * k > delta)


def test_rd_equals_split_bitwise(orc):
    """For P a power of two, the canonical tree makes all algorithms return
    bit-identical values (reading R-8)."""
    for P in [2, 4, 8]:
        for k in [1000, 3000]:          # sparse throughout / densifies midway
            streams = synth.uniform_streams(P, 20000, k, seed=P, kind="normal")
            a, _ = orc.ssar_recursive_double(20000, streams)
            b, _, _ = orc.split_allgather(20000, streams, algo=orc.ALGO_SSAR_SPLIT)
            ma, va = orc.result_to_dense(a[0], 20000)
            mb, vb = orc.result_to_dense(b[0], 20000)
            np.testing.assert_array_equal(va.view(np.uint32), vb.view(np.uint32))
            if not a[0][0] and not b[0][0]:
                np.testing.assert_array_equal(a[0][1], b[0][1])


def test_dsar_phase2_volume(orc):
    """DSAR phase 2 moves exactly (P-1)/P*N values per rank."""
    for P, N in [(2, 4096), (4, 4096), (8, 65536)]:
        streams = synth.uniform_streams(P, N, N // 4, seed=P, kind="int")
        res, st, dsar = orc.split_allgather(N, streams, algo=orc.ALGO_DSAR_SPLIT)
        assert dsar
        # phase-1 received bytes are 8 per pair; subtract them
        _, st_ssar, _ = orc.split_allgather(N, streams, algo=orc.ALGO_SSAR_SPLIT)
        for r in range(P):
            part = N // P
            ph1 = sum(8 * int(np.count_nonzero((streams[i][0] >= r * part) & (streams[i][0] < (r + 1) * part)))
                      for i in range(P) if i != r)
            assert st[r]["bytes_recv"] - ph1 == 4 * (P - 1) * N // P


def test_dsar_quantized_volume(orc):
    P, N, bits, B = 8, 65536, 4, 1024
    streams = synth.uniform_streams(P, N, N // 4, seed=3, kind="int")
    _, st_q, _ = orc.split_allgather(N, streams, algo=orc.ALGO_DSAR_SPLIT, quant_bits=bits, bucket=B)
    _, st_f, _ = orc.split_allgather(N, streams, algo=orc.ALGO_DSAR_SPLIT)
    part = N // P
    per = (part * bits + 7) // 8 + 4 * ((part + B - 1) // B)
    for r in range(P):
        assert st_f[r]["bytes_recv"] - st_q[r]["bytes_recv"] == (P - 1) * (4 * part - per)


def test_split_nonuniform_partition(orc):
    """N not divisible by P: floor(N/P) per rank, remainder on the last."""
    P, N = 3, 100
    streams = [(np.arange(N, dtype=np.uint32), np.ones(N, np.float32))] * P
    res, st, _ = orc.split_allgather(N, streams, algo=orc.ALGO_SSAR_SPLIT, delta=N)
    np.testing.assert_array_equal(res[0][2], np.full(N, 3.0, np.float32))
    # owner 2 holds 100 - 2*33 = 34 coordinates: phase 1 brings 2 slices of 34
    # pairs, phase 2 brings R_0 and R_1 of 33 pairs each
    assert st[2]["bytes_recv"] == 2 * 34 * 8 + 2 * 33 * 8
    assert st[0]["bytes_recv"] == 2 * 33 * 8 + (33 + 34) * 8


def test_dsar_quantized_decodes_within_bound(orc):
    """DSAR + QSGD: every coordinate is within scale/s of the exact sum."""
    P, N, bits = 4, 8192, 4
    streams = synth.uniform_streams(P, N, 2000, seed=5, kind="normal")
    res, _, _ = orc.split_allgather(N, streams, algo=orc.ALGO_DSAR_SPLIT, quant_bits=bits, bucket=1024, seed=9)
    mask, acc, _ = _dense_ref(N, streams)
    exact = acc.astype(np.float32)
    s = 2 ** (bits - 1) - 1
    for b in range(N // 1024):
        sl = slice(b * 1024, (b + 1) * 1024)
        scale = np.abs(exact[sl]).max()
        assert np.all(np.abs(res[0][2][sl] - exact[sl]) <= scale / s * (1 + 1e-6) + 1e-6)
    for r in range(1, P):
        np.testing.assert_array_equal(res[r][2], res[0][2])


# ---- sparse allgather for disjoint slices (§7 SCD; reading R-27) ---------

def _slices(P, N, per, seed, order=None):
    """Rank r's `per` indices inside its own slice of the model vector."""
    rng = np.random.default_rng(seed)
    bounds = np.linspace(0, N, P + 1).astype(np.int64)
    order = list(range(P)) if order is None else order
    streams = []
    for r in range(P):
        s = order[r]
        lo, hi = bounds[s], bounds[s + 1]
        n = min(per, hi - lo)
        i = np.sort(rng.choice(np.arange(lo, hi), n, replace=False)).astype(np.uint32)
        streams.append((i, rng.standard_normal(n).astype(np.float32)))
    return streams


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
def test_sparse_allgather_equals_definition(orc, P):
    """Disjoint slices: the allgather is the union, i.e. the brute-force sum
    (one contributor per index) -- any mistake in ordering, offsets or values
    shows up against the independent dense definition."""
    N = 10_000
    rng = np.random.default_rng(P)
    order = list(rng.permutation(P))             # slices owned in a shuffled rank order
    streams = _slices(P, N, 100, seed=P, order=order)
    res, st = orc.sparse_allgather(N, streams)
    bf = orc.brute_force(N, streams)
    for r in range(P):
        d, i, v = res[r]
        assert not d
        np.testing.assert_array_equal(i, np.nonzero(bf["mask"])[0])
        np.testing.assert_array_equal(v, bf["f32"][i])
        n_r = len(streams[r][0])
        assert st[r]["bytes_recv"] == 8 * (sum(len(s[0]) for s in streams) - n_r)
        assert st[r]["bytes_sent"] == 8 * n_r * (P - 1)


def test_sparse_allgather_dense_and_empty(orc):
    N, P = 1000, 4
    streams = _slices(P, N, 200, seed=1)          # K = 800 > delta = 500: dense
    streams[2] = (np.zeros(0, np.uint32), np.zeros(0, np.float32))
    res, _ = orc.sparse_allgather(N, streams)
    bf = orc.brute_force(N, streams)
    d, _, v = res[0]
    assert d
    np.testing.assert_array_equal(v, bf["f32"])


def test_sparse_allgather_rejects_overlapping_ranges(orc):
    a = (np.array([1, 50], np.uint32), np.ones(2, np.float32))
    b = (np.array([10, 20], np.uint32), np.ones(2, np.float32))   # inside a's range
    with pytest.raises(ValueError):
        orc.sparse_allgather(100, [a, b])


# ---- recursive doubling for non-power-of-two P (App. A; reading R-28) -----------

@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("P", [3, 5, 6, 7, 12])
def test_rd_folded_matches_definition(orc, seed, P):
    """Folding the extra ranks in and out around recursive doubling still
    computes the definition (integer values: exactly; normal values: within
    the rounding bound), on every rank including the extra ones."""
    rng = np.random.default_rng(7000 + 10 * P + seed)
    N = int(rng.choice([500, 4096]))
    d = float(rng.choice([0.01, 0.1, 0.3]))
    k = max(1, int(d * N))
    kind = "int" if seed % 2 == 0 else "normal"
    streams = synth.uniform_streams(P, N, k, seed=seed, kind=kind)
    res, st = orc.ssar_recursive_double(N, streams)
    _check_against_definition(N, streams, res, kind == "int", orc.switch_threshold(N))


def test_rd_folded_order_and_volume(orc):
    """P = 3: the tree is (x0 + x2) + x1 -- pinned with values whose fp32 sums
    differ by order -- and the extra rank sends its stream once and receives
    the result once."""
    N = 8
    big, tiny = np.float32(1.0), np.float32(2.0 ** -24)
    x0 = (np.array([0], np.uint32), np.array([big], np.float32))
    x1 = (np.array([0], np.uint32), np.array([tiny], np.float32))
    x2 = (np.array([0], np.uint32), np.array([tiny], np.float32))
    res, st = orc.ssar_recursive_double(N, [x0, x1, x2])
    want = np.float32(np.float32(big + tiny) + tiny)          # (x0 + x2) + x1, round to nearest even
    for r in range(3):
        d, i, v = res[r]
        assert not d and list(i) == [0] and v[0] == want
    assert st[2]["bytes_sent"] == 8 and st[2]["bytes_recv"] == 8 and st[2]["msgs_sent"] == 1
    assert st[0]["bytes_recv"] == 8 + 8 and st[0]["bytes_sent"] == 8 + 8   # fold in + RD stage, RD stage + result out
    assert st[1]["bytes_sent"] == 8 and st[1]["bytes_recv"] == 8


# ---- MAX / MIN operators (§5: any associative op with a neutral element) ---------

@pytest.mark.parametrize("op", [1, 2])
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_max_min_all_algorithms_equal_definition(orc, op, P):
    """MAX and MIN are associative and commutative, so every algorithm must
    return exactly the definition: on the union the op over the holders, and
    the neutral element (-inf / +inf) where a dense result has no entry."""
    for N, k in [(4096, 40), (4096, 1500)]:          # stays sparse / switches to dense
        streams = synth.uniform_streams(P, N, k, seed=op * 10 + P, kind="normal")
        mask, want = orc.brute_force_op(N, streams, op)
        with orc.op_scope(op):
            results = [orc.ssar_recursive_double(N, streams)[0]]
            for algo in (orc.ALGO_SSAR_SPLIT, orc.ALGO_DSAR_SPLIT):
                results.append(orc.split_allgather(N, streams, algo=algo)[0])
        for res in results:
            for d, i, v in res:
                if d:
                    np.testing.assert_array_equal(v, want)
                    assert np.all(np.isinf(v[mask == 0]))
                else:
                    np.testing.assert_array_equal(i, np.nonzero(mask)[0])
                    np.testing.assert_array_equal(v, want[i])
        # MAX of a set >= every member, MIN <= (the definition is not SUM)
        vals = np.full((P, N), np.nan, np.float32)
        for r, (i, v) in enumerate(streams):
            vals[r, i] = v
        sel = ~np.all(np.isnan(vals), 0)
        ref = np.zeros(N, np.float32)
        ref[sel] = np.nanmax(vals[:, sel], 0) if op == 1 else np.nanmin(vals[:, sel], 0)
        np.testing.assert_array_equal(want[mask == 1], ref[mask == 1])


def test_quantization_requires_sum(orc):
    streams = synth.uniform_streams(2, 4096, 100, seed=1)
    with orc.op_scope(1):
        with pytest.raises(ValueError):
            orc.split_allgather(4096, streams, algo=orc.ALGO_DSAR_SPLIT, quant_bits=4)


# ---- DSAR + QSGD: every element of the N-vector draws its own Philox counter ----------

@pytest.mark.parametrize("P,N,B", [(2, 4096, 256), (4, 8192, 1024), (8, 8192, 512)])
def test_dsar_qsgd_counter_is_the_global_index(orc, P, N, B):
    """partition j's QSGD draws use ctr_base = b_j, so the
    element at global index g draws u(seed, g).  Input: the dense sum is 1 at
    every bucket start and 1/2 elsewhere (integer-free but exact: 1/4 + 1/4),
    at 2 bits (s = 1) a 1/2 decodes to 1 iff u >= 1/2 iff bit 31 of Philox
    word g%4 of counter g/4 is set -- computed from the KAT-pinned Philox
    block, not from the quantizer.  A counter base of 0 per partition (every
    owner reusing one stream) fails for every partition j >= 1."""
    seed = 12345
    idx = np.arange(N, dtype=np.uint32)
    v = np.full(N, 0.25, np.float32)
    v[::B] = 0.5
    streams = [(idx, v), (idx, v)] + [(np.zeros(0, np.uint32), np.zeros(0, np.float32))] * (P - 2)
    res, _, used = orc.split_allgather(N, streams, algo=orc.ALGO_DSAR_SPLIT, quant_bits=2, bucket=B, seed=seed)
    out = res[0][2]
    key = np.array([seed & 0xFFFFFFFF, seed >> 32], np.uint32)
    expect = np.empty(N, np.float32)
    for c in range(N // 4):
        w = orc.philox4x32_10(np.array([c, 0, 0, 0], np.uint32), key)
        for q in range(4):
            expect[4 * c + q] = 1.0 if (w[q] >> 31) else 0.0
    expect[::B] = 1.0            # |v| = scale decodes exactly (level s)
    np.testing.assert_array_equal(out, expect)
    for r in range(1, P):
        np.testing.assert_array_equal(res[r][2], out)
