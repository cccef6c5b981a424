"""Stress driver (torchrun, one rank per GPU): hundreds of back-to-back
collectives on one IPC world, cycling algorithms, operators, sizes and
collectives without host synchronisation between them, every result checked
against the oracle.  Catches flag/sequence races that single calls cannot.
Run: python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tests/stress_worker.py [iters]"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1802_08021_b200 import sparcml as S  # noqa: E402
from paper_1802_08021_b200 import synth  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    N0, kmax = 60_000, 12_000
    comm = S.Comm(200_000, 60_000)
    rng = np.random.default_rng(1234)   # same sequence of cases on every rank
    # auto_big: split-allgather with the SSAR/DSAR decision left to the device;
    # *64: fp64 values
    kinds = ["rd", "ssar", "dsar", "dsar4", "allgather", "max", "auto", "auto_big", "rd64", "ssar64", "dsar64"]
    pending, fails = [], 0
    for it in range(iters):
        kind = kinds[int(rng.integers(len(kinds)))]
        N = 200_000 if kind == "auto_big" else N0
        f64 = kind.endswith("64")
        base = kind[:-2] if f64 else ("auto" if kind == "auto_big" else kind)
        k = int(rng.integers(0, 60_000 if kind == "auto_big" else kmax))
        seed = int(rng.integers(1 << 30))
        if kind == "allgather":
            bounds = np.linspace(0, N, P + 1).astype(np.int64)
            order = np.random.default_rng(seed).permutation(P)
            streams = []
            for r in range(P):
                lo, hi = bounds[order[r]], bounds[order[r] + 1]
                n = min(k // P, hi - lo)
                g = np.random.default_rng(seed + r)
                streams.append((np.sort(g.choice(np.arange(lo, hi), n, replace=False)).astype(np.uint32),
                                g.standard_normal(n).astype(np.float32)))
        else:
            streams = synth.uniform_streams(P, N, k, seed=seed, kind="normal64" if f64 else "normal")
        i, v = streams[rank]
        it_ = torch.from_numpy(i.view(np.int32)).cuda()
        vt = torch.from_numpy(v).cuda()
        if kind == "allgather":
            out = comm.allgather(it_, vt, N)
        else:
            algo = {"rd": S.SSAR_RECURSIVE_DOUBLE, "ssar": S.SSAR_SPLIT_ALLGATHER, "dsar": S.DSAR_SPLIT_ALLGATHER,
                    "dsar4": S.DSAR_SPLIT_ALLGATHER, "max": S.SSAR_SPLIT_ALLGATHER, "auto": S.ALGO_AUTO}[base]
            opts = S.make_opts(algo=algo, quant_bits=4 if kind == "dsar4" else 0, seed=seed & 0xFFFF)
            out = comm.allreduce(it_, vt, N, opts=opts, op=S.OP_MAX if kind == "max" else S.OP_SUM)
        pending.append((base, streams, out, seed, it_, vt, N, np.float64 if f64 else np.float32))
        if len(pending) >= 8 or it == iters - 1:   # check in batches: calls run back to back on the device
            torch.cuda.synchronize()
            for kind, streams, out, seed, _, _, N, dt in pending:
                g = S.read_result(out)
                if kind == "allgather":
                    ref, _ = oracle.sparse_allgather(N, streams)
                elif kind == "max":
                    with oracle.op_scope(oracle.OP_MAX):
                        ref, _, _ = oracle.split_allgather(N, streams, algo=oracle.ALGO_SSAR_SPLIT)
                elif kind == "rd":
                    ref, _ = oracle.ssar_recursive_double(N, streams, dtype=dt)
                else:
                    a = {"ssar": oracle.ALGO_SSAR_SPLIT, "dsar": oracle.ALGO_DSAR_SPLIT, "dsar4": oracle.ALGO_DSAR_SPLIT,
                         "auto": oracle.ALGO_AUTO}[kind]
                    ref, _, _ = oracle.split_allgather(N, streams, algo=a, quant_bits=4 if kind == "dsar4" else 0,
                                                       seed=seed & 0xFFFF, dtype=dt)   # AUTO: split at every size
                d, ei, ev = ref[rank]
                ok = g.header.status == 0 and g.dense == d
                if ok and d:
                    ok = np.array_equal(g.val.cpu().numpy(), ev)
                elif ok:
                    ok = np.array_equal(g.idx.cpu().numpy().view(np.uint32), ei) and np.array_equal(g.val.cpu().numpy(), ev)
                if not ok:
                    fails += 1
                    print(f"rank {rank}: {kind} MISMATCH (status {g.header.status})", flush=True)
            pending = []
    t = torch.tensor([fails])
    dist.all_reduce(t)
    comm.close()
    if rank == 0:
        print(f"stress P={P} iters={iters}: {'OK' if t.item() == 0 else 'FAILED'} ({int(t.item())} mismatches)", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if t.item() == 0 else 1)


if __name__ == "__main__":
    main()
