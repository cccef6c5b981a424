"""Pins for the App. B result-size analysis: the paper's
inclusion-exclusion sum against the binomial-theorem closed form
N(1-(1-d)^P), the cited values, the union bound, and Monte Carlo over
exactly-k uniform supports including the measured K of a real allreduce."""
import json
import os

import numpy as np
import pytest

from paper_1802_08021_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_cited_values(orc):
    with open(os.path.join(GOLD, "expected_nnz.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        assert abs(orc.expected_nnz(c["k"], c["N"], c["P"]) - c["E"]) < 1e-9 * max(1, c["E"]), c["cite"]


@pytest.mark.parametrize("P", [1, 2, 3, 8, 16, 32])
def test_closed_form_and_union_bound(orc, P):
    for N in [512, 4096, 2 ** 24]:
        for k in [1, N // 100, N // 10, N // 2, N]:
            e = orc.expected_nnz(k, N, P)
            cf = N * (1.0 - (1.0 - k / N) ** P)
            assert abs(e - cf) <= 1e-9 * N
            assert e <= min(N, P * k) + 1e-6


def test_monte_carlo_and_measured(orc):
    """Config 1 (P=4, N=4096, k=64): E[K] = 250.06; sample K over seeds
    (through the RD simulator) within 3 standard errors of the mean."""
    P, N, k = 4, 4096, 64
    Ks = []
    for s in range(400):
        res, _ = orc.ssar_recursive_double(N, synth.uniform_streams(P, N, k, seed=s))
        Ks.append(len(res[0][1]))
    Ks = np.array(Ks, np.float64)
    e = orc.expected_nnz(k, N, P)
    assert abs(Ks.mean() - e) < 3 * Ks.std() / np.sqrt(len(Ks))
