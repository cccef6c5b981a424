"""Algorithm 1 training a synthetic sparse logistic regression
(config 5's data structure, NEXT row 2) on a loopback world: every rank
computes its gradient at the current model on the GPU (plumbing, torch ops),
then the hot path -- EF top-k, sparse allreduce, v <- v - g -- runs in the
library.  Each step is bit-exact against the same step composed from oracle
pieces fed the same gradients, and the loss goes down."""
import numpy as np
import pytest

from paper_1802_08021_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1802_08021_b200 import sparcml as S  # noqa: E402


def lr_grad_loss(w, feat, y):
    """Mean logistic loss and its gradient for binary features (duplicates in a row count once)."""
    X = torch.zeros(feat.shape[0], w.numel(), device=w.device)
    X.scatter_(1, feat, 1.0)
    m = X @ w
    loss = torch.nn.functional.binary_cross_entropy_with_logits(m, y)
    g = X.t() @ (torch.sigmoid(m) - y) / feat.shape[0]
    return loss.item(), g.contiguous()


@pytest.mark.parametrize("P,bucket", [(4, 0), (3, 512)])
def test_lr_training_matches_oracle_and_learns(orc, P, bucket):
    N, samples, feats, steps, alpha = 20_000, 256, 20, 12, 2.0
    k = 200 if bucket == 0 else 8
    data = synth.lr_dataset(P, N, samples=samples, feats=feats, seed=3)
    dev = [(torch.from_numpy(f).cuda(), torch.from_numpy(y).cuda()) for f, y in data]
    kk = S.topk_count(N, k, bucket)
    w = S.LocalWorld(P, N, kk)
    v_d = [torch.zeros(N, device="cuda") for _ in range(P)]
    e_d = [torch.zeros(N, device="cuda") for _ in range(P)]
    v_h = [np.zeros(N, np.float32) for _ in range(P)]
    e_h = [np.zeros(N, np.float32) for _ in range(P)]
    opts = S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER)
    losses = []
    for step in range(steps):
        gl = [lr_grad_loss(v_d[r], *dev[r]) for r in range(P)]
        losses.append(float(np.mean([x[0] for x in gl])))
        grads = [x[1] for x in gl]
        grads_h = [g.cpu().numpy() for g in grads]
        streams = [S.ef_topk(e_d[r], grads[r], alpha, k, bucket=bucket) for r in range(P)]
        outs = w.allreduce(streams, N, opts=opts)
        for r in range(P):
            S.apply_update(v_d[r], outs[r])
        hs = []
        for r in range(P):
            if bucket:
                i, v, e_h[r] = orc.ef_topk_bucketed(e_h[r], grads_h[r], alpha, k, bucket)
            else:
                i, v, e_h[r] = orc.ef_topk(e_h[r], grads_h[r], alpha, k)
            hs.append((i, v))
        ref, _, _ = orc.split_allgather(N, hs, algo=orc.ALGO_SSAR_SPLIT)
        for r in range(P):
            v_h[r] = orc.apply_update(v_h[r], ref[r], N)   # v <- v - g
            np.testing.assert_array_equal(e_d[r].cpu().numpy(), e_h[r])
            np.testing.assert_array_equal(v_d[r].cpu().numpy(), v_h[r])
        for r in range(1, P):   # every rank applies the same g: the replicas stay identical
            assert torch.equal(v_d[r], v_d[0])
    assert losses[0] == pytest.approx(np.log(2.0), abs=1e-6)   # w = 0
    assert losses[-1] < losses[0] - 0.02, losses
