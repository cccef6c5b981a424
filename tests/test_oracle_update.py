"""Pins for the oracle's Algorithm-1 update v <- v - g (or_apply_update):
a hand-worked example, the dense/sparse equivalence, untouched coordinates
bit-for-bit, one fp32 rounding per touched coordinate, and fp64."""
import numpy as np
import pytest

from paper_1802_08021_b200 import synth


def test_worked_example(orc):
    v = np.array([1.0, 2.0, 3.0, 4.0], np.float32)
    res = (False, np.array([1, 3], np.uint32), np.array([0.5, -1.0], np.float32))
    np.testing.assert_array_equal(orc.apply_update(v, res, 4), [1.0, 1.5, 3.0, 5.0])
    dense = (True, None, np.array([1.0, 1.0, 0.0, -2.0], np.float32))
    np.testing.assert_array_equal(orc.apply_update(v, dense, 4), [0.0, 1.0, 3.0, 6.0])


def test_absent_coordinates_untouched_and_signed_zero_kept(orc):
    v = np.array([-0.0, 7.0, np.float32(1e-30), 2.0], np.float32)
    out = orc.apply_update(v, (False, np.array([3], np.uint32), np.array([2.0], np.float32)), 4)
    assert np.signbit(out[0]) and out[1] == 7.0 and out[2] == np.float32(1e-30) and out[3] == 0.0


def test_one_rounding_per_coordinate(orc):
    """fl(1 - 2^-25) = 1 (one rounding, tie-free); two half-updates would differ."""
    v = np.ones(2, np.float32)
    out = orc.apply_update(v, (False, np.array([0], np.uint32), np.array([2.0 ** -25], np.float32)), 2)
    assert out[0] == 1.0
    out = orc.apply_update(v, (False, np.array([0], np.uint32), np.array([2.0 ** -24], np.float32)), 2)
    assert out[0] == np.float32(1.0 - 2.0 ** -24)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_sparse_equals_dense_scatter(orc, dtype):
    N = 5000
    rng = np.random.default_rng(4)
    idx = np.sort(rng.choice(N, 700, replace=False)).astype(np.uint32)
    g = rng.standard_normal(700).astype(dtype)
    v = rng.standard_normal(N).astype(dtype)
    gd = np.zeros(N, dtype)
    gd[idx] = g
    a = orc.apply_update(v, (False, idx, g), N, dtype=dtype)
    b = orc.apply_update(v, (True, None, gd), N, dtype=dtype)
    np.testing.assert_array_equal(a, b)
    ref = v.copy()
    ref[idx] = ref[idx] - g        # numpy's elementwise IEEE subtraction, one rounding
    np.testing.assert_array_equal(a, ref)


def test_out_of_range_index_is_an_error(orc):
    with pytest.raises(ValueError):
        orc.apply_update(np.zeros(4, np.float32), (False, np.array([4], np.uint32), np.ones(1, np.float32)), 4)
