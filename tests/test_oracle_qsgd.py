"""Pins for the oracle's QSGD codec (§6) and its Philox RNG:
Random123 known-answer vectors, cited examples, exact packing, the exact
size formula, boundedness |dec - v| <= scale/s, and unbiasedness within 3
standard errors (the defining property of stochastic quantization)."""
import json
import os

import numpy as np
import pytest

from paper_1802_08021_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_philox_kat(orc):
    for v in _load("philox_kat.json")["vectors"]:
        ctr = [int(h, 16) for h in v["ctr"]]
        key = [int(h, 16) for h in v["key"]]
        out = orc.philox4x32_10(ctr, key)
        assert [f"{w:08x}" for w in out] == v["out"]


def test_uniform_draws(orc):
    us = np.array([orc.qsgd_uniform(5, c) for c in range(40000)])
    assert us.min() >= 0.0 and us.max() < 1.0
    assert abs(us.mean() - 0.5) < 3 * np.sqrt(1 / 12 / len(us))
    # the draw for counter c is word c%4 of block c//4
    w = orc.philox4x32_10([3, 0, 0, 0], [5, 0])
    assert orc.qsgd_uniform(5, 14) == (int(w[2]) >> 8) / 2.0 ** 24


def test_examples(orc):
    ex = _load("qsgd_examples.json")
    x = np.array(ex["round_trip_at_scale"]["x"], np.float32)
    for b in ex["round_trip_at_scale"]["bits"]:
        c, s = orc.qsgd_quantize(x, b, bucket=1024, seed=1)
        np.testing.assert_array_equal(orc.qsgd_dequantize(c, s, len(x), b, 1024), x)
    z = np.array(ex["zero_bucket"]["x"], np.float32)
    c, s = orc.qsgd_quantize(z, 4)
    assert np.all(c == 0) and np.all(s == 0)
    d = orc.qsgd_dequantize(c, s, 4, 4)
    assert np.all(d == 0) and not np.any(np.signbit(d))
    e = ex["level_s_scale_3"]
    c, s = orc.qsgd_quantize(np.array(e["x"], np.float32), e["bits"], seed=3)
    np.testing.assert_array_equal(orc.qsgd_dequantize(c, s, 4, e["bits"])[:2], e["decoded_first"])
    p = ex["packing"]
    c, s = orc.qsgd_quantize(np.array(p["x"], np.float32), p["bits"], bucket=p["bucket"], seed=0)
    assert c.tobytes().hex() == p["codes_hex"]
    np.testing.assert_array_equal(s, p["scales"])


def test_half_probability(orc):
    h = _load("qsgd_examples.json")["half_probability"]
    n = h["trials"]
    x = np.tile(np.array(h["x"], np.float32), n)        # buckets of 2: [1.0, 0.5]
    c, s = orc.qsgd_quantize(x, h["bits"], bucket=2, seed=11)
    d = orc.qsgd_dequantize(c, s, len(x), h["bits"], 2)
    assert np.all(d[0::2] == 1.0)
    assert set(np.unique(d[1::2])) <= {0.0, 1.0}
    assert abs(d[1::2].mean() - h["mean"]) < h["tol"]


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("B", [4, 100, 1024])
def test_size_and_bound(orc, bits, B):
    x = synth.gaussian_vector(3001, seed=bits + B)
    c, s = orc.qsgd_quantize(x, bits, bucket=B, seed=2, ctr_base=12345)
    assert len(c) == (3001 * bits + 7) // 8 and len(s) == (3001 + B - 1) // B
    d = orc.qsgd_dequantize(c, s, 3001, bits, B)
    lv = 2 ** (bits - 1) - 1
    for b in range(len(s)):
        sl = slice(b * B, min((b + 1) * B, 3001))
        assert s[b] == np.abs(x[sl]).max()
        assert np.all(np.abs(d[sl] - x[sl]) <= s[b] / lv * (1 + 2 ** -20))
        assert np.all(np.abs(d[sl]) <= s[b])
    assert np.all(np.sign(d[d != 0]) == np.sign(x[d != 0]))


def test_unbiased(orc):
    """E[dequantize(quantize(v))] = v: mean over 2000 seeds within 3 SE."""
    x = synth.gaussian_vector(64, seed=9)
    T = 2000
    acc = np.zeros(64)
    acc2 = np.zeros(64)
    for t in range(T):
        c, s = orc.qsgd_quantize(x, 4, bucket=64, seed=t)
        d = orc.qsgd_dequantize(c, s, 64, 4, 64).astype(np.float64)
        acc += d
        acc2 += d * d
    mean = acc / T
    var = acc2 / T - mean ** 2
    se = np.sqrt(np.maximum(var, 1e-30) / T)
    z = np.abs(mean - x) / se
    assert np.mean(z < 3) > 0.97 and np.all(z < 5)


def test_counter_base_shifts_stream(orc):
    x = synth.gaussian_vector(2048, seed=1)
    c1, _ = orc.qsgd_quantize(x[1024:], 4, seed=7, ctr_base=1024)
    c2, _ = orc.qsgd_quantize(x, 4, seed=7, ctr_base=0)
    np.testing.assert_array_equal(c1, c2[512:])


# ---- l2-norm scale (reading R-31) ------------------------------------------------------

@pytest.mark.parametrize("B", [8, 64, 1024])
def test_l2_scale_is_the_bucket_norm(orc, B):
    """The l2 scale is the bucket's Euclidean norm (numpy, fp64) to fp32
    accuracy, every decoded magnitude is <= it, and a bucket holding a single
    non-zero value has scale = |value| exactly (the tree adds only zeros)."""
    x = synth.gaussian_vector(3001, seed=B)
    with orc.qsgd_norm_scope(1):
        c, s = orc.qsgd_quantize(x, 4, bucket=B, seed=3)
        d = orc.qsgd_dequantize(c, s, len(x), 4, B)
        for b in range(len(s)):
            sl = slice(b * B, min((b + 1) * B, len(x)))
            ref = np.sqrt(np.sum(x[sl].astype(np.float64) ** 2))
            assert abs(float(s[b]) - ref) <= 2e-6 * ref
            assert np.all(np.abs(d[sl]) <= s[b])
        one = np.zeros(B, np.float32)
        one[B // 3] = np.float32(-3.75)
        _, s1 = orc.qsgd_quantize(one, 8, bucket=B, seed=1)
        assert s1[0] == np.float32(3.75)


def test_l2_unbiased(orc):
    """E[dequantize(quantize(v))] = v with the l2 scale too (within 3 SE)."""
    x = synth.gaussian_vector(64, seed=19)
    T = 2000
    acc = np.zeros(64)
    acc2 = np.zeros(64)
    with orc.qsgd_norm_scope(1):
        for t in range(T):
            c, s = orc.qsgd_quantize(x, 4, bucket=64, seed=t)
            d = orc.qsgd_dequantize(c, s, 64, 4, 64).astype(np.float64)
            acc += d
            acc2 += d * d
    mean = acc / T
    var = acc2 / T - mean ** 2
    se = np.sqrt(np.maximum(var, 1e-30) / T)
    z = np.abs(mean - x) / se
    assert np.mean(z < 3) > 0.97 and np.all(z < 5)


def test_l2_needs_power_of_two_bucket(orc):
    with orc.qsgd_norm_scope(1):
        with pytest.raises(ValueError):
            orc.qsgd_quantize(np.ones(10, np.float32), 4, bucket=100)


def test_l2_scale_summation_order_is_the_adjacent_pair_tree(orc):
    """Pins the ORDER of R-31's sum of squares, not only its value: hand-derived
    inputs on which the balanced adjacent-pair tree, a sequential fold, a
    reversed fold and a strided tree all round differently (tests/golden)."""
    g = _load("qsgd_examples.json")["l2_tree_order"]
    ulp = np.float32(2.0 ** -23)
    small = np.float32(2.0 ** -12)
    for case in g["cases"]:
        B = case["B"]
        x = np.zeros(B, np.float32)
        x[0] = 1.0
        if B == 64:
            x[1:] = small
        else:
            x[4:] = small
        with orc.qsgd_norm_scope(1):
            _, s = orc.qsgd_quantize(x, 8, bucket=B, seed=0)
        assert s[0] == np.float32(1.0) + np.float32(case["scale_minus_1_in_ulps"]) * ulp, (B, s[0])
