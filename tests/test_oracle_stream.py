"""Pins for the oracle's sparse-stream layer (§5.1).

Each oracle function is checked against something other than itself: the
worked examples (tests/golden/stream_examples.json, cited), and brute force
with numpy's dense scatter-add on small random inputs (the plain definition
of a coordinate-wise sum)."""
import json
import os

import numpy as np
import pytest

from paper_1802_08021_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _pairs(lst):
    if not lst:
        return np.zeros(0, np.uint32), np.zeros(0, np.float32)
    a = np.array(lst, dtype=np.float64)
    return a[:, 0].astype(np.uint32), a[:, 1].astype(np.float32)


def test_switch_threshold_examples(orc):
    for ex in _load("stream_examples.json")["switch_threshold"]:
        assert orc.switch_threshold(ex["N"], ex["isize"], ex["c"]) == ex["delta"], ex["cite"]


def test_switch_threshold_definition(orc):
    # delta is the largest nnz for which nnz*(c+isize) <= N*isize
    for N in [1, 2, 3, 7, 100, 4096, 2**24, 25_557_032]:
        for isize, c in [(4, 4), (8, 4), (4, 3), (8, 3)]:
            d = orc.switch_threshold(N, isize, c)
            assert d * (c + isize) <= N * isize < (d + 1) * (c + isize)
    assert orc.switch_threshold(1000, 4, 4, 0.5) == 250


def test_merge_examples(orc):
    for ex in _load("stream_examples.json")["merge_sum"]:
        ia, va = _pairs(ex["a"])
        ib, vb = _pairs(ex["b"])
        io, vo = orc.merge_sum(ia, va, ib, vb)
        eo, ev = _pairs(ex["out"])
        np.testing.assert_array_equal(io, eo)
        np.testing.assert_array_equal(vo, ev)


def test_dense_switch_example(orc):
    ex = _load("stream_examples.json")["dense_switch"]
    delta = orc.switch_threshold(ex["N"], ex["isize"], ex["c"])
    assert delta == 5
    ia, va = _pairs(ex["a"])
    ib, vb = _pairs(ex["b"])
    d, i, v = orc.stream_sum(ex["N"], delta, (False, ia, va), (False, ib, vb))
    assert d is True
    np.testing.assert_array_equal(v, np.array(ex["dense_out"], np.float32))
    assert int(np.count_nonzero(v)) == 6


def _dense_ref(N, streams):
    """numpy brute force: scatter-add every stream into a zero vector."""
    acc = np.zeros(N, np.float64)
    mask = np.zeros(N, bool)
    for idx, val in streams:
        np.add.at(acc, idx.astype(np.int64), val.astype(np.float64))
        mask[idx] = True
    return mask, acc


@pytest.mark.parametrize("seed", range(6))
def test_merge_matches_brute_force(orc, seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 300))
    ka, kb = int(rng.integers(0, N + 1)), int(rng.integers(0, N + 1))
    (ia, va), (ib, vb) = synth.uniform_streams(2, N, [ka, kb], seed=seed, kind="int")
    io, vo = orc.merge_sum(ia, va, ib, vb)
    mask, acc = _dense_ref(N, [(ia, va), (ib, vb)])
    np.testing.assert_array_equal(io, np.nonzero(mask)[0])
    np.testing.assert_array_equal(vo.astype(np.float64), acc[io])   # integer values: exact
    assert np.all(np.diff(io.astype(np.int64)) > 0)                   # strictly increasing


@pytest.mark.parametrize("case", ["ss_sparse", "ss_dense", "sd", "ds", "dd"])
def test_stream_sum_four_cases(orc, case):
    N = 97
    (ia, va), (ib, vb) = synth.uniform_streams(2, N, [30, 40], seed=3, kind="int")
    da = np.zeros(N, np.float32); da[ia] = va
    db = np.zeros(N, np.float32); db[ib] = vb
    if case == "ss_sparse":
        d, i, v = orc.stream_sum(N, 70, (False, ia, va), (False, ib, vb))
        assert not d
        mask, acc = _dense_ref(N, [(ia, va), (ib, vb)])
        np.testing.assert_array_equal(i, np.nonzero(mask)[0])
        np.testing.assert_array_equal(v, acc[i].astype(np.float32))
        return
    if case == "ss_dense":
        d, i, v = orc.stream_sum(N, 69, (False, ia, va), (False, ib, vb))   # 30+40 > 69
    elif case == "sd":
        d, i, v = orc.stream_sum(N, 48, (False, ia, va), (True, None, db))
    elif case == "ds":
        d, i, v = orc.stream_sum(N, 48, (True, None, da), (False, ib, vb))
    else:
        d, i, v = orc.stream_sum(N, 48, (True, None, da), (True, None, db))
    assert d
    np.testing.assert_array_equal(v, da + db)


def test_brute_force_definition(orc):
    streams = synth.uniform_streams(3, 50, [10, 20, 5], seed=1, kind="normal")
    bf = orc.brute_force(50, streams)
    mask, acc = _dense_ref(50, streams)
    np.testing.assert_array_equal(bf["mask"].astype(bool), mask)
    np.testing.assert_allclose(bf["d64"], acc, rtol=0, atol=1e-12)
    assert bf["K"] == int(mask.sum())
    seq = np.zeros(50, np.float32)
    for idx, val in streams:             # fp32 left fold in rank order
        for j, x in zip(idx, val):
            seq[j] = np.float32(seq[j] + x)
    np.testing.assert_array_equal(bf["f32"], seq)
