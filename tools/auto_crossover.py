"""Measure the recursive-doubling vs split-allgather crossover on this box
(§8.1: recursive doubling is best for small data),
one rank per GPU:

  python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/auto_crossover.py

For N in 2^12 .. 2^24 and densities 1/16 .. 1/256 (uniform supports, exactly k
per rank) both algorithms run as CUDA graphs, 20 timed replays each after a
device barrier, max over ranks.  Rank 0 prints one JSON line per point and a
summary: the largest sum_i k_i * 8 bytes at which recursive doubling still
wins (the table compiled into AUTO, csrc/api.cu kRdMaxBytes).
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_08021_b200 import sparcml as S, synth  # noqa: E402


def main():
    dist.init_process_group("cpu:gloo,cuda:nccl")
    rank, P = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    maxN = 1 << 24
    comm = S.Comm(maxN, maxN // 16)
    rows = []
    for lgN in range(12, 25, 2):
        N = 1 << lgN
        for dd in (16, 64, 256):
            k = max(1, N // dd)
            i, v = synth.uniform_streams(P, N, k, seed=lgN + dd)[rank]
            it = torch.from_numpy(i.view(np.int32)).cuda()
            vt = torch.from_numpy(v).cuda()
            out = S.new_out(N)
            res = {}
            for name, algo in (("rd", S.SSAR_RECURSIVE_DOUBLE), ("split", S.SSAR_SPLIT_ALLGATHER)):
                opts = S.make_opts(algo=algo, k_sum_hint=P * k)
                for _ in range(3):
                    comm.barrier()
                    comm.allreduce(it, vt, N, out=out, opts=opts)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    comm.allreduce(it, vt, N, out=out, opts=opts)
                ts = []
                for _ in range(20):
                    comm.barrier()
                    torch.cuda._sleep(200000)
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record()
                    g.replay()
                    b.record()
                    b.synchronize()
                    ts.append(a.elapsed_time(b) * 1e3)
                t = torch.tensor([float(np.median(ts))], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                res[name] = float(t.item())
                assert S.read_result(out).header.status == 0
            row = {"P": P, "N": N, "k": k, "ksum_bytes": 8 * P * k, "rd_us": res["rd"], "split_us": res["split"]}
            rows.append(row)
            if rank == 0:
                print(json.dumps(row), flush=True)
    if rank == 0:
        win = [r["ksum_bytes"] for r in rows if r["rd_us"] < r["split_us"]]
        lose = [r["ksum_bytes"] for r in rows if r["rd_us"] >= r["split_us"]]
        print(json.dumps({"P": P, "rd_wins_max_ksum_bytes": max(win) if win else 0,
                          "split_wins_min_ksum_bytes": min(lose) if lose else None}), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
