"""Stand-alone union-merge-with-sum (sparcml_merge_sum, §5.1): CUDA-event
time per launch (L2 flushed before each) and the HBM fraction of SURVEY §8(d)'s
algorithmic bytes 8(na + nb) + 8 n_out (diagnostics; bench.py reports the same
number as merge_roofline).

  python tools/merge_bench.py [--N 16777216] [--density 0.1] [--reps 20]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_08021_b200 import sparcml as S, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1 << 24)
ap.add_argument("--density", type=float, default=0.10)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
dev = torch.device("cuda", 0)
N = args.N
k = synth.k_for_density(N, args.density)
(ia, va), (ib, vb) = synth.uniform_streams(2, N, k, seed=7)
cu = lambda a: torch.from_numpy(a).to(dev)
ia, va, ib, vb = cu(ia.view("int32")), cu(va), cu(ib.view("int32")), cu(vb)
io = torch.empty(2 * k, dtype=torch.int32, device=dev)
vo = torch.empty(2 * k, dtype=torch.float32, device=dev)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
wsb = int(S._lib.sparcml_ops_workspace_bytes(2 * k))
ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def run():
    S._check(S._lib.sparcml_merge_sum(ia.data_ptr(), va.data_ptr(), k, ib.data_ptr(), vb.data_ptr(), k,
                                      io.data_ptr(), vo.data_ptr(), cnt.data_ptr(), ws.data_ptr(), wsb,
                                      S._stream(None)))


for _ in range(3):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(args.reps):
    flush.zero_()
    flush.view(torch.int64).sum()
    torch.cuda._sleep(200000)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
n_out = int(cnt.item())
if "marks" in os.environ.get("SPARCML_LIB", ""):
    ws[64:256].zero_()
    torch.cuda.synchronize()
    flush.zero_()
    t0 = torch.cuda.Event(enable_timing=True)
    run()
    torch.cuda.synchronize()
    mk = ws[64:256].cpu().numpy().view(np.uint64).astype(np.float64)
    base = mk[0]
    names = ["start", "searched", "staged", "merged", "looked-back", "written"]
    print("block 0 first chunk (us): " + ", ".join(f"{n} {(mk[i] - base) / 1e3:.2f}" for i, n in enumerate(names)))
    print("latest chunk (us):        " + ", ".join(f"{n} {(mk[12 + i] - base) / 1e3:.2f}" for i, n in enumerate(names)))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.1)
alg = 8 * 2 * k + 8 * n_out
t = float(np.median(ts))
print(f"merge 2 x {k} -> {n_out}: us per launch median {t:.2f} min {min(ts):.2f}; {alg / t / 1e3:.1f} GB/s, "
      f"frac {alg / t / 1e3 / peak:.3f} of {peak} GB/s")
