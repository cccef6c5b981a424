"""Sparse allgather for disjoint slices (§7 SCD; reading R-27)
on loopback worlds against the oracle: every rank's result is the union of
the ranks' streams in range order, bit-exact (no arithmetic), with the
oracle's byte accounting; overlapping ranges are reported in the header."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1802_08021_b200 import sparcml as S  # noqa: E402


def slices(P, N, per, seed, empty=()):
    rng = np.random.default_rng(seed)
    bounds = np.linspace(0, N, P + 1).astype(np.int64)
    order = rng.permutation(P)
    out = []
    for r in range(P):
        lo, hi = bounds[order[r]], bounds[order[r] + 1]
        n = 0 if r in empty else min(per, hi - lo)
        i = np.sort(rng.choice(np.arange(lo, hi), n, replace=False)).astype(np.uint32)
        out.append((i, rng.standard_normal(n).astype(np.float32)))
    return out


def cuda(streams):
    return [(torch.from_numpy(i.view(np.int32)).cuda(), torch.from_numpy(v).cuda()) for i, v in streams]


@pytest.mark.parametrize("P,N,per,empty", [(1, 1000, 100, ()), (2, 100_000, 100, ()), (3, 1 << 20, 5000, (1,)),
                                           (5, 77_777, 777, ()), (8, 1 << 20, 100, (0, 7)),
                                           (4, 4000, 700, ()), (16, 65_536, 1000, ())])
def test_allgather_matches_oracle(orc, P, N, per, empty):
    streams = slices(P, N, per, seed=P * 13 + N, empty=empty)
    w = S.LocalWorld(P, N, max(1, per))
    outs = w.allgather(cuda(streams), N)
    ref, st = orc.sparse_allgather(N, streams)
    for r in range(P):
        g = S.read_result(outs[r])
        d, ei, ev = ref[r]
        assert g.header.status == 0 and g.header.algo_used == S.SPARSE_ALLGATHER
        assert g.dense == bool(d)
        if d:
            np.testing.assert_array_equal(g.val.cpu().numpy(), ev)
        else:
            np.testing.assert_array_equal(g.idx.cpu().numpy().view(np.uint32), ei)
            np.testing.assert_array_equal(g.val.cpu().numpy(), ev)
        assert g.header.bytes_recv == st[r]["bytes_recv"] and g.header.bytes_sent == st[r]["bytes_sent"]
    # repeated calls on the same world
    outs2 = w.allgather(cuda(streams), N)
    a, b = S.read_result(outs[0]), S.read_result(outs2[-1])
    assert a.header.nnz == b.header.nnz and a.dense == b.dense
    np.testing.assert_array_equal(a.val.cpu().numpy(), b.val.cpu().numpy())


def test_allgather_overlap_reported():
    a = (np.array([1, 50], np.uint32), np.ones(2, np.float32))
    b = (np.array([10, 20], np.uint32), np.ones(2, np.float32))
    w = S.LocalWorld(2, 100, 2)
    outs = w.allgather(cuda([a, b]), 100)
    assert S.read_result(outs[0]).header.status == S.ERR_INVALID_ARG
    # the next call with valid input is clean again
    c = (np.array([60, 70], np.uint32), np.ones(2, np.float32))
    outs = w.allgather(cuda([a, c]), 100)
    assert S.read_result(outs[1]).header.status == 0
