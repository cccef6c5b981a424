"""NCCL bus bandwidth on this box (ncclAllGather and pairwise
send/recv busbw at 256 MB - 1 GB), one rank per GPU:

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/nccl_busbw.py

busbw conventions of nccl-tests: allgather (P-1)/P * total bytes / t,
allreduce 2(P-1)/P * bytes / t, send/recv bytes / t (ranks 0 <-> 1, each
direction at once).  CUDA events, best of 5 after 2 warm-ups; rank 0 prints
one JSON line (diagnostics; the bench reads profiles/nvlink_peak.json).
"""
import json
import os

import torch
import torch.distributed as dist


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        t = torch.tensor([a.elapsed_time(b) / 1e3], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        best = min(best, float(t.item()))
    return best


def main():
    dist.init_process_group("nccl")
    rank, P = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    out = {"P": P, "allgather": [], "allreduce": [], "sendrecv": []}
    for mb in (256, 1024):
        n = (mb << 20) // 4
        x = torch.ones(n, device="cuda")
        y = torch.empty(n * P, device="cuda")
        t = timed(lambda: dist.all_gather_into_tensor(y, x))
        out["allgather"].append({"bytes_per_rank": 4 * n, "busbw_gbs": (P - 1) / P * 4 * n * P / t / 1e9})
        t = timed(lambda: dist.all_reduce(x))
        out["allreduce"].append({"bytes": 4 * n, "busbw_gbs": 2 * (P - 1) / P * 4 * n / t / 1e9})
        if P >= 2:
            r = torch.empty(n, device="cuda")

            def sr():
                if rank in (0, 1):
                    peer = 1 - rank
                    ops = [dist.P2POp(dist.isend, x, peer), dist.P2POp(dist.irecv, r, peer)]
                    for q in dist.batch_isend_irecv(ops):
                        q.wait()
            t = timed(sr)
            out["sendrecv"].append({"bytes": 4 * n, "per_direction_gbs": 4 * n / t / 1e9})
        del x, y
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
