"""Algorithm 1 training synthetic sparse logistic regression on
one process per GPU: each rank computes its gradient at the current model
(torch ops), then the library's hot path runs -- EF top-k, the sparse
allreduce over NVLink, v <- v - g (sparcml.algorithm1_step).  Prints the mean
loss per step (rank 0).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 examples/lr_algorithm1.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_08021_b200 import sparcml as S  # noqa: E402
from paper_1802_08021_b200 import synth  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    N, samples, feats, steps, k, bucket = 200_000, 1000, 50, 40, 2000, 0
    alpha = 1.0 / P   # Algorithm 1 sums the P sparsified updates
    feat, y = synth.lr_dataset(P, N, samples=samples, feats=feats, seed=1)[rank]
    feat, y = torch.from_numpy(feat).cuda(), torch.from_numpy(y).cuda()
    X = torch.zeros(samples, N, device="cuda")
    X.scatter_(1, feat, 1.0)
    comm = S.Comm(N, S.topk_count(N, k, bucket))
    v = torch.zeros(N, device="cuda")
    eps = torch.zeros(N, device="cuda")
    opts = S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER)
    for step in range(steps):
        m = X @ v
        loss = torch.nn.functional.binary_cross_entropy_with_logits(m, y)
        grad = (X.t() @ (torch.sigmoid(m) - y) / samples).contiguous()
        out = S.algorithm1_step(comm, v, eps, grad, alpha, k, bucket=bucket, opts=opts)
        t = torch.tensor([loss.item()])
        dist.all_reduce(t)
        if rank == 0:
            h = S.read_result(out).header
            print(f"step {step:3d}  mean loss {t.item() / P:.5f}  |g| nnz {h.nnz}  algo {h.algo_used}", flush=True)
    vs = [torch.zeros(1)] * P
    dist.all_gather_object(vs, float(v.double().sum().item()))
    if rank == 0:
        print("replicas identical:", len(set(vs)) == 1, flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
