"""Global EF top-k on one GPU: CUDA-event time per launch (L2 flushed before
each) and, with a marks-enabled library, the per-phase %globaltimer breakdown
(diagnostics; numbers under a profiler or with marks are not bench values).

  python tools/topk_phases.py [--N 16777216] [--density 0.01] [--reps 20] [--plain]
  SPARCML_LIB=/tmp/lib_marks.so python tools/topk_phases.py        (phase marks)

Phases (kernels_topk.cu, tk_mark): 0 start (CTA 0) | 1 sample done | 2 filter
done | 3 barrier A released | 4 range located | 5 barrier B released |
6 offsets known | 7 placement done (each the latest CTA's time).
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_08021_b200 import sparcml as S, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1 << 24)
ap.add_argument("--density", type=float, default=0.01)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--plain", action="store_true", help="plain top-k (no EF)")
ap.add_argument("--pre", type=int, default=5, help="untimed calls first (EF: the accumulator settles, warm start)")
ap.add_argument("--noflush", action="store_true", help="skip the L2 flush between launches (diagnostics)")
args = ap.parse_args()
N = args.N
k = max(1, int(args.density * N))
dev = torch.device("cuda", 0)
g = torch.from_numpy(synth.gaussian_vector(N, seed=0)).to(dev)
eps = torch.zeros(N, device=dev)
ws = S.TopkWorkspace(N, k, dev)
io = torch.empty(k, dtype=torch.int32, device=dev)
vo = torch.empty(k, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
marks = "marks" in os.environ.get("SPARCML_LIB", "")


def run():
    if args.plain:
        S.topk_sparsify(g, k, ws=ws, idx_out=io, val_out=vo)
    else:
        S.ef_topk(eps, g, 0.01, k, ws=ws, idx_out=io, val_out=vo)


for _ in range(args.pre):
    run()
torch.cuda.synchronize()
ts, ph, tcs = [], [], []
for _ in range(args.reps):
    if not args.noflush:
        flush.zero_()
        flush.view(torch.int64).sum()
    ws.buf[56:56 + 128 + 256].zero_()
    torch.cuda._sleep(200000)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
    if marks:
        t = ws.buf[56:56 + 128].cpu().numpy().view(np.uint64).astype(np.float64)
        d = ws.buf[184:184 + 256].cpu().numpy().view(np.uint64).astype(np.float64)
        raw = ws.buf[184 + 160:184 + 224].cpu().numpy().view(np.uint64).copy()
        TC = 205248
        G = 148
        tc = ws.buf[TC:TC + 2 * 1024 * 8].cpu().numpy().view(np.uint64).reshape(2, 1024)[:, :G].astype(np.float64)
        tcs.append(((tc[0] - t[0]) / 1e3, (tc[1] - t[0]) / 1e3))
        d = np.where(d > 0, (d - t[0]) / 1e3, np.nan)
        if not np.isfinite(d[11]) or not np.isfinite(d[8]):
            pass
        ph.append(np.concatenate([(t[1:8] - t[0]) / 1e3, [(t[8] - t[0]) / 1e3], (t[9:15] - t[0]) / 1e3, d[:21]]))
st = ws.status()
ts = np.array(ts)
alg = (12 if not args.plain else 4) * N + 8 * k
print(f"N={N} k={k} {'plain' if args.plain else 'EF'}: us per launch median {np.median(ts):.2f} "
      f"p25 {np.percentile(ts, 25):.2f} p75 {np.percentile(ts, 75):.2f} min {ts.min():.2f}; "
      f"alg bytes {alg} -> {alg / np.median(ts) / 1e3:.1f} GB/s; status {st}")
if ph:
    p = np.nanmedian(np.array(ph), axis=0)
    names = ["sample", "filter", "barrierA", "locate", "barrierB", "offsets", "place"]
    print("phase ends, latest CTA (us after CTA 0 starts, median): " + ", ".join(f"{n} {v:.2f}" for n, v in zip(names, p)))
    print(f"latest CTA start {p[7]:.2f}; CTA 0 phase ends: " + ", ".join(f"{n} {v:.2f}" for n, v in zip(names, p[8:14])))
 
    st0 = np.median(np.array([x[0] for x in tcs]), axis=0)
    fe = np.median(np.array([x[1] for x in tcs]), axis=0)
    print("per-CTA start p0/p50/p100 %.2f %.2f %.2f; filter end p0/p10/p50/p90/p100 %.2f %.2f %.2f %.2f %.2f" % (
        st0.min(), np.median(st0), st0.max(), fe.min(), np.percentile(fe, 10), np.median(fe), np.percentile(fe, 90), fe.max()))
    print("CTA 0 values: tau %x split %x cta_n %d fast_ok %d crossing cnt %d bin %d fast %d kth %x" % tuple(int(v) for v in raw))
    print("CTA 0 fine marks (TK_D 0..20): " + " ".join(f"{i}:{v:.2f}" for i, v in enumerate(p[14:])))
