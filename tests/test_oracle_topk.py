"""Pins for the oracle's top-k and error feedback (§2.2 P:216-224,
Algorithm 1): cited examples, brute force against numpy's lexsort
(a library routine) with forced ties, exact reconstruction and magnitude
dominance invariants, and the Algorithm-1 degenerate case."""
import json
import os

import numpy as np
import pytest

from paper_1802_08021_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_topk_examples(orc):
    with open(os.path.join(GOLD, "topk_examples.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        i, v, r = orc.topk(np.array(c["x"], np.float32), c["k"], residual=True)
        np.testing.assert_array_equal(i, c["idx"], err_msg=c["cite"])
        np.testing.assert_array_equal(v, np.array(c["val"], np.float32), err_msg=c["cite"])
        np.testing.assert_array_equal(r, np.array(c["residual"], np.float32), err_msg=c["cite"])


def _lexsort_topk(x, k):
    order = np.lexsort((np.arange(len(x)), -np.abs(x.astype(np.float64))))
    sel = np.sort(order[:min(k, len(x))])
    return sel


@pytest.mark.parametrize("seed", range(10))
def test_topk_brute_force_with_ties(orc, seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 5000))
    # few distinct magnitudes -> many ties at the k-th value
    x = (rng.integers(-6, 7, size=N) * 0.25).astype(np.float32)
    k = int(rng.integers(1, N + 2))
    i, v, r = orc.topk(x, k, residual=True)
    sel = _lexsort_topk(x, k)
    np.testing.assert_array_equal(i, sel)
    np.testing.assert_array_equal(v, x[sel])
    # reconstruction: selected + residual == input exactly
    rec = r.copy()
    rec[i] += v
    np.testing.assert_array_equal(rec, x)
    # dominance
    if 0 < len(i) < N:
        rest = np.delete(np.abs(x), i)
        assert np.abs(v).min() >= rest.max()


def test_topk_gaussian(orc):
    x = synth.gaussian_vector(100_000, seed=4)
    k = 100
    i, v = orc.topk(x, k)
    np.testing.assert_array_equal(i, _lexsort_topk(x, k))
    assert np.all(np.diff(i.astype(np.int64)) > 0)


def test_ef_degenerate_sgd(orc):
    """P=1, k=N, Q=identity: every coordinate is sent, eps stays 0 and the
    sent values are alpha*grad (Algorithm 1)."""
    g = synth.gaussian_vector(1000, seed=1)
    eps = np.zeros(1000, np.float32)
    i, v, e = orc.ef_topk(eps, g, 0.125, 1000)       # alpha a power of 2: exact
    np.testing.assert_array_equal(i, np.arange(1000))
    np.testing.assert_array_equal(v, np.float32(0.125) * g)
    assert np.all(e == 0)


def test_ef_accumulates(orc):
    """acc = eps + alpha*g, eps <- acc - TopK(acc).  Dyadic values keep every
    operation exact so fmaf and the two-rounding form agree."""
    rng = np.random.default_rng(7)
    N, k = 512, 17
    eps = (rng.integers(-64, 64, size=N) / 16).astype(np.float32)
    g = (rng.integers(-64, 64, size=N) / 8).astype(np.float32)
    alpha = 0.5
    i, v, e = orc.ef_topk(eps, g, alpha, k)
    acc = eps.astype(np.float64) + alpha * g.astype(np.float64)
    sel = _lexsort_topk(acc.astype(np.float32), k)
    np.testing.assert_array_equal(i, sel)
    np.testing.assert_array_equal(v, acc[sel].astype(np.float32))
    want = acc.copy()
    want[sel] = 0
    np.testing.assert_array_equal(e, want.astype(np.float32))
    # conservation of gradient mass over steps: sum(sent) + eps == sum(alpha*g)
    eps2, sent = np.zeros(N, np.float32), np.zeros(N, np.float64)
    for step in range(5):
        gs = (rng.integers(-64, 64, size=N) / 8).astype(np.float32)
        i, v, eps2 = orc.ef_topk(eps2, gs, 0.5, k)
        sent[i] += v
        if step == 0:
            total = 0.5 * gs.astype(np.float64)
        else:
            total += 0.5 * gs.astype(np.float64)
    np.testing.assert_array_equal(sent + eps2, total)


# ---- bucketed top-k (§7; reading R-26) -------------------

def _lexsort_bucketed(x, k, B):
    out = []
    for b0 in range(0, len(x), B):
        out.append(b0 + _lexsort_topk(x[b0:b0 + B], k))
    return np.concatenate(out) if out else np.zeros(0, np.int64)


@pytest.mark.parametrize("seed", range(8))
def test_topk_bucketed_brute_force_with_ties(orc, seed):
    """Per bucket against numpy's lexsort (a library routine), ragged last
    bucket, forced ties, k above and below the bucket size."""
    rng = np.random.default_rng(100 + seed)
    N = int(rng.integers(1, 6000))
    B = int(rng.choice([1, 3, 128, 512, 1000, 4096]))
    k = int(rng.integers(1, min(B, 40) + 2))
    x = (rng.integers(-6, 7, size=N) * 0.25).astype(np.float32)
    i, v, r = orc.topk_bucketed(x, k, B, residual=True)
    sel = _lexsort_bucketed(x, k, B)
    np.testing.assert_array_equal(i, sel)
    np.testing.assert_array_equal(v, x[sel])
    assert len(i) == orc.bucketed_count(N, k, B) == sum(min(k, len(x[b:b + B])) for b in range(0, N, B))
    rec = r.copy()
    rec[i] += v
    np.testing.assert_array_equal(rec, x)
    # dominance inside every bucket
    for b0 in range(0, N, B):
        ib = i[(i >= b0) & (i < b0 + B)] - b0
        xb = np.abs(x[b0:b0 + B])
        if 0 < len(ib) < len(xb):
            assert xb[ib].min() >= np.delete(xb, ib).max()


def test_topk_bucketed_special_cases(orc):
    x = synth.gaussian_vector(10_000, seed=11)
    # one bucket covering the vector is the global top-k
    i1, v1 = orc.topk_bucketed(x, 77, 1 << 20)
    i2, v2 = orc.topk(x, 77)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(v1, v2)
    # k >= B keeps everything; B = 1 with k = 1 keeps everything
    for k, B in [(512, 512), (600, 512), (1, 1)]:
        i, v = orc.topk_bucketed(x, k, B)
        np.testing.assert_array_equal(i, np.arange(len(x)))
        np.testing.assert_array_equal(v, x)
    # the paper's setting: 4 of every 512 -> 4 per full bucket
    i, _ = orc.topk_bucketed(x, 4, 512)
    assert len(i) == 19 * 4 + 4
    assert np.all(np.bincount(i // 512, minlength=20) == 4)


def test_ef_topk_bucketed_matches_definition(orc):
    rng = np.random.default_rng(9)
    N, k, B = 3000, 5, 512
    eps = (rng.integers(-64, 64, size=N) / 16).astype(np.float32)
    g = (rng.integers(-64, 64, size=N) / 8).astype(np.float32)
    i, v, e = orc.ef_topk_bucketed(eps, g, 0.5, k, B)
    acc = (eps.astype(np.float64) + 0.5 * g.astype(np.float64)).astype(np.float32)   # exact (dyadic)
    sel = _lexsort_bucketed(acc, k, B)
    np.testing.assert_array_equal(i, sel)
    np.testing.assert_array_equal(v, acc[sel])
    want = acc.copy()
    want[sel] = 0
    np.testing.assert_array_equal(e, want)
