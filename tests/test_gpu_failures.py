"""Failure handling ("every rank calls with the same arguments in
the same order"; SURVEY §5 failure detection), on loopback worlds with the
library's failure injection:

* a dead rank (its kernels never launch): every flag wait of the others gives
  up after the communicator's timeout, the call completes and the waiting
  ranks' headers report SPARCML_ERR_TIMEOUT -- no hang;
* a rank calling with another signature (N / op / algo / options): the call
  signature travels with every exchange and every rank's header reports
  SPARCML_ERR_MISMATCH (recursive doubling propagates it along the stages);
* back-to-back sparse allgathers on one world stay correct (the published
  streams alternate by call parity).
"""
import time

import numpy as np
import pytest

from paper_1802_08021_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1802_08021_b200 import sparcml as S  # noqa: E402


def cuda_streams(streams):
    return [(torch.from_numpy(i.view(np.int32)).cuda(), torch.from_numpy(v).cuda()) for i, v in streams]


def _disjoint(P, N, per, seed):
    rng = np.random.default_rng(seed)
    part = N // P
    out = []
    for r in range(P):
        idx = np.sort(rng.choice(part, per, replace=False)).astype(np.uint32) + np.uint32(r * part)
        out.append((idx, rng.standard_normal(per).astype(np.float32)))
    return out


@pytest.mark.parametrize("algo,P", [(S.SSAR_SPLIT_ALLGATHER, 2), (S.SSAR_SPLIT_ALLGATHER, 4),
                                    (S.DSAR_SPLIT_ALLGATHER, 4), (S.SSAR_RECURSIVE_DOUBLE, 2),
                                    (S.SSAR_RECURSIVE_DOUBLE, 4), (S.SSAR_RECURSIVE_DOUBLE, 3)])
def test_dead_rank_times_out(algo, P):
    N, k = 1 << 16, 500
    w = S.LocalWorld(P, N, k)
    w.set_timeout(150)
    w.inject(S.INJECT_SKIP_RANKS, 1 << (P - 1))      # the last rank is dead
    st = cuda_streams(synth.uniform_streams(P, N, k, seed=3))
    t0 = time.time()
    outs = w.allreduce(st, N, opts=S.make_opts(algo=algo))
    torch.cuda.synchronize()
    assert time.time() - t0 < 30
    stats = [S.read_result(outs[r]).header.status for r in range(P - 1)]
    assert S.ERR_TIMEOUT in stats, stats
    if algo != S.SSAR_RECURSIVE_DOUBLE:   # split: every live owner waits for the dead source
        assert all(s == S.ERR_TIMEOUT for s in stats), stats
    w.close()


def test_dead_rank_times_out_allgather():
    P, N = 3, 30_000
    w = S.LocalWorld(P, N, 1000)
    w.set_timeout(150)
    w.inject(S.INJECT_SKIP_RANKS, 0b010)
    outs = w.allgather(cuda_streams(_disjoint(P, N, 300, seed=1)), N)
    torch.cuda.synchronize()
    assert [S.read_result(outs[r]).header.status for r in (0, 2)] == [S.ERR_TIMEOUT, S.ERR_TIMEOUT]
    w.close()


@pytest.mark.parametrize("algo,P,bad", [(S.SSAR_SPLIT_ALLGATHER, 2, 1), (S.SSAR_SPLIT_ALLGATHER, 4, 2),
                                        (S.DSAR_SPLIT_ALLGATHER, 4, 0), (S.SSAR_RECURSIVE_DOUBLE, 2, 0),
                                        (S.SSAR_RECURSIVE_DOUBLE, 4, 3), (S.SSAR_RECURSIVE_DOUBLE, 8, 5),
                                        (S.SSAR_RECURSIVE_DOUBLE, 6, 5)])
def test_mismatched_rank_reported_everywhere(algo, P, bad):
    N, k = 1 << 16, 400
    w = S.LocalWorld(P, N, k)
    st = cuda_streams(synth.uniform_streams(P, N, k, seed=5))
    outs = w.allreduce(st, N, opts=S.make_opts(algo=algo))       # a clean call first
    assert all(S.read_result(o).header.status == 0 for o in outs)
    w.inject(S.INJECT_PERTURB_SIG, bad + 1)
    outs = w.allreduce(st, N, opts=S.make_opts(algo=algo))
    torch.cuda.synchronize()
    assert [S.read_result(o).header.status for o in outs] == [S.ERR_MISMATCH] * P
    w.inject(S.INJECT_PERTURB_SIG, 0)                              # and clean again
    outs = w.allreduce(st, N, opts=S.make_opts(algo=algo))
    assert all(S.read_result(o).header.status == 0 for o in outs)
    w.close()


def test_mismatched_rank_allgather():
    P, N = 4, 40_000
    w = S.LocalWorld(P, N, 1000)
    w.inject(S.INJECT_PERTURB_SIG, 3)
    outs = w.allgather(cuda_streams(_disjoint(P, N, 200, seed=2)), N)
    torch.cuda.synchronize()
    assert [S.read_result(o).header.status for o in outs] == [S.ERR_MISMATCH] * P
    w.close()


def test_injection_is_loopback_only_and_checked():
    w = S.LocalWorld(2, 1000, 10)
    with pytest.raises(S.SparcmlError):
        w.inject(99, 1)
    w.close()


def test_back_to_back_allgathers(orc):
    """Many allgathers in a row on one world, changing inputs every call."""
    P, N = 4, 80_000
    w = S.LocalWorld(P, N, 2000)
    for it in range(12):
        streams = _disjoint(P, N, 100 + 37 * it, seed=10 + it)
        outs = w.allgather(cuda_streams(streams), N)
        ref, _ = orc.sparse_allgather(N, streams)
        for r in range(P):
            res = S.read_result(outs[r])
            assert res.header.status == 0
            d, ei, ev = ref[r]
            np.testing.assert_array_equal(res.idx.cpu().numpy().view(np.uint32), ei)
            np.testing.assert_array_equal(res.val.cpu().numpy(), ev)
    w.close()
