"""DSAR owner (densify + canonical-tree reduce + QSGD, the a6/a7 rows) at
config 4's sizes on a loopback world: per-launch time of dsar_owner_kernel from
the library's event bracket (L2 flushed before each call), and the whole
allreduce.  Diagnostics; `--ncu` runs a few calls only (for an ncu capture).

  python tools/dsar_owner_bench.py [--P 4] [--bits 4] [--reps 10]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_08021_b200 import sparcml as S, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=4)
ap.add_argument("--bits", type=int, default=4)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--N", type=int, default=1 << 24)
args = ap.parse_args()
P, N = args.P, args.N
k = synth.k_for_density(N, 0.10)
st = synth.uniform_streams(P, N, k, seed=4)
streams = [(torch.from_numpy(i.view(np.int32)).cuda(), torch.from_numpy(v).cuda()) for i, v in st]
w = S.LocalWorld(P, N, k)
outs = [S.new_out(N) for _ in range(P)]
opts = S.make_opts(algo=S.DSAR_SPLIT_ALLGATHER, quant_bits=args.bits, seed=3)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    w.allreduce(streams, N, outs=outs, opts=opts)
torch.cuda.synchronize()
S.profile_reset()
S.profile_only(None)
ts = []
for _ in range(args.reps):
    flush.zero_()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    S.profile_enable(True)
    a.record()
    w.allreduce(streams, N, outs=outs, opts=opts)
    b.record()
    S.profile_enable(False)
    b.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
res = S.read_result(outs[0])
prof = {n: S.profile_read(n) for n in S.PROFILED_KERNELS}
prof = {n: (c, ms) for n, (c, ms) in prof.items() if c}
n_own, ms_own = prof.get("owner_dsar", (0, 0.0))
part = N // P
print(f"P={P} N={N} k={k} bits={args.bits}: loopback allreduce {np.median(ts):.1f} us (all {P} ranks' kernels), "
      f"status {res.header.status}, dense {res.dense}")
if n_own:
    t = ms_own / n_own * 1e3
    alg = 8 * (P * k) / P + (part * args.bits + 7) // 8 + 4 * ((part + 1023) // 1024) if args.bits else 8 * k + 4 * part
    print(f"dsar_owner: {t:.1f} us per launch over {n_own} launches; {part} positions per owner -> "
          f"{t * 1e3 / part:.2f} ns per position; alg bytes {alg} -> {alg / t / 1e3:.1f} GB/s")
print({n: round(ms / c * 1e3, 1) for n, (c, ms) in prof.items()})
