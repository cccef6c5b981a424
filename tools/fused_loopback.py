"""The fused split-allgather kernel on a loopback world (all P ranks on one
GPU, the same kernel and protocol as one rank per GPU) at config 2's sizes:
diagnostics and a single-GPU ncu target.

  python tools/fused_loopback.py [--P 4] [--reps 20] [--ncu]
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
ap.add_argument("--N", type=int, default=1 << 24)
ap.add_argument("--density", type=float, default=0.01)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--ncu", action="store_true", help="a few calls only")
args = ap.parse_args()
P, N = args.P, args.N
k = int(args.density * N)
st = synth.uniform_streams(P, N, k, seed=1)
streams = [(torch.from_numpy(i.view(np.int32)).cuda(), torch.from_numpy(v).cuda()) for i, v in st]
w = S.LocalWorld(P, N, k)
outs = [S.new_out(N) for _ in range(P)]
opts = S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER)
reps = 3 if args.ncu else args.reps
for _ in range(3):
    w.allreduce(streams, N, outs=outs, opts=opts)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    w.allreduce(streams, N, outs=outs, opts=opts)
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
h = S.read_result(outs[0]).header
print(f"P={P} N={N} k={k} fused={os.environ.get('SPARCML_FUSED', '1')}: loopback allreduce median {np.median(ts):.1f} us "
      f"(all {P} ranks on one GPU); status {h.status} nnz {h.nnz}")
