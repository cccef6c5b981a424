"""Algorithm 1, the full training step, on a loopback world:
acc = eps + alpha*grad; eps <- acc - TopK(acc); g = allreduce(Q(TopK(acc)), SUM);
v <- v - g -- with Q = identity and Q = QSGD on the selected values (reading
R-29), global and bucketed selection, over three steps of carried
state, bit-exact against the same step composed from oracle pieces."""
import numpy as np
import pytest

from paper_1802_08021_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1802_08021_b200 import sparcml as S  # noqa: E402


@pytest.mark.parametrize("P,N,k,bucket,qbits", [(4, 100_000, 1000, 0, 0), (3, 65_536, 4, 512, 0),
                                                 (4, 200_003, 2000, 0, 4), (2, 1 << 18, 8, 512, 8)])
def test_algorithm1_steps_match_oracle(orc, P, N, k, bucket, qbits):
    alpha, seed, qb = 0.05, 11, 512
    kk = S.topk_count(N, k, bucket)
    w = S.LocalWorld(P, N, kk)
    v_h = [np.zeros(N, np.float32) for _ in range(P)]
    e_h = [np.zeros(N, np.float32) for _ in range(P)]
    v_d = [torch.zeros(N, device="cuda") for _ in range(P)]
    e_d = [torch.zeros(N, device="cuda") for _ in range(P)]
    opts = S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER)
    for step in range(3):
        grads = [synth.gaussian_vector(N, seed=step, rank=r) for r in range(P)]
        # device: the step, rank by rank (the allreduce is the loopback collective)
        streams = []
        for r in range(P):
            i, v = S.ef_topk(e_d[r], torch.from_numpy(grads[r]).cuda(), alpha, k, bucket=bucket)
            if qbits:
                c, sc = S.quantize(v, qbits, bucket=qb, seed=seed, ctr_base=r * kk)
                v = S.dequantize(c, sc, v.numel(), qbits, bucket=qb)
            streams.append((i, v))
        outs = w.allreduce(streams, N, opts=opts)
        for r in range(P):
            S.apply_update(v_d[r], outs[r])
        # oracle: the same step from its pieces
        hs = []
        for r in range(P):
            if bucket:
                i, v, e_h[r] = orc.ef_topk_bucketed(e_h[r], grads[r], alpha, k, bucket)
            else:
                i, v, e_h[r] = orc.ef_topk(e_h[r], grads[r], alpha, k)
            if qbits:
                c, sc = orc.qsgd_quantize(v, qbits, bucket=qb, seed=seed, ctr_base=r * kk)
                v = orc.qsgd_dequantize(c, sc, len(v), qbits, qb)
            hs.append((i, v))
        ref, _, _ = orc.split_allgather(N, hs, algo=orc.ALGO_SSAR_SPLIT)
        for r in range(P):
            v_h[r] = orc.apply_update(v_h[r], ref[r], N)   # v <- v - g
            np.testing.assert_array_equal(e_d[r].cpu().numpy(), e_h[r])
            np.testing.assert_array_equal(v_d[r].cpu().numpy(), v_h[r])
