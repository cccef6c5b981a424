#!/usr/bin/env python
"""bench.py — SparCML hot path on B200: EF top-k + sparse allreduce.

One step (default workload, BASELINE.json configs[1]) per rank:
  ef_topk  : acc = eps + alpha*grad, k = 1% of N = 2^24 largest |acc|
             (top-k of an i.i.d. Gaussian gradient = a uniform-random support
             of exactly k indices, the paper's micro-benchmark input P:937-938)
  allreduce: SSAR_Split_allgather of the P streams over NVLink (CUDA IPC)
value = whole-job "effective GB/s": dense-equivalent bytes reduced per second,
        P * 4N / t_step.  ms_per_step is the step latency.

Timing: W warm-up steps, then K steps, each bracketed by CUDA events on the
launching stream; L2 is flushed (512 MiB write, then read back clean) before every step outside the
events; barrier + synchronize around the timed region; max over ranks.

Launch: python bench.py [--gpus N --steps K --warmup W] ; N > 1 under
torchrun (one rank per GPU).  --impl reference times the CPU oracle instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse allreduce latency (µs) and effective GB/s at N, density, 1/2/4/8 B200"

CONFIGS = {
    "cfg2": dict(desc="BASELINE configs[1]: N=16M (2^24) fp32, density 1% uniform-random support per rank "
                      "(EF top-k of a Gaussian gradient), SSAR_Split_allgather",
                 N=1 << 24, density=0.01, algo="ssar_split", bits=0),
    "cfg3": dict(desc="BASELINE configs[2]: top-k 0.1% of a 25,557,032-parameter Gaussian gradient, "
                      "SSAR_Recursive_double",
                 N=25_557_032, density=0.001, algo="rd", bits=0),
    "cfg4": dict(desc="BASELINE configs[3]: N=2^24, density 10%, DSAR_Split_allgather with QSGD 4-bit",
                 N=1 << 24, density=0.10, algo="dsar", bits=4),
    # the paper's DNN selector, k of every bucket of 512
    "bucket512": dict(desc="NEXT (SURVEY 8f rank 2): bucketed EF top-k, 4 of every 512 (P:1238), of a "
                           "25,557,032-parameter Gaussian gradient, SSAR_Split_allgather",
                      N=25_557_032, density=4 / 512, algo="ssar_split", bits=0, bucket=512, kb=4),
}


def step_k(cfg, N=None):
    """(k passed to top-k, entries it writes)."""
    N = cfg["N"] if N is None else N
    if cfg.get("bucket"):
        B, kb = cfg["bucket"], cfg["kb"]
        full, tail = divmod(N, B)
        return kb, full * min(kb, B) + (min(kb, tail) if tail else 0)
    k = max(1, int(cfg["density"] * N))
    return k, k


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["sparcml", "reference"], default="sparcml")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


# A ~0.5 ms spin kernel ahead of each timed step: the start event then fires
# when the GPU reaches the step, not while it idles waiting for the host to
# finish enqueueing (host launch latency is not kernel time; e2e keeps it).
HOLD_CYCLES = 1_000_000   # ~0.5 ms: covers host jitter (e.g. the clock sampler) while the step is enqueued


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str):
    """dram read+write bytes per launch of `kernel` from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["kernels"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, dev: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU oracle leg (reference arm and cpu_baseline): plain single-threaded C
# ---------------------------------------------------------------------------
def oracle_step_time(cfg, P_sim, N_s, seed=0):
    """One step of the workload at dimension N_s for P_sim ranks on the CPU
    oracle (EF top-k per rank + the collective simulation).  Returns seconds."""
    import numpy as np
    import oracle
    from paper_1802_08021_b200 import synth
    k, _ = step_k(cfg, N_s)
    grads = [synth.gaussian_vector(N_s, seed=seed, rank=r) for r in range(P_sim)]
    eps = [np.zeros(N_s, np.float32) for _ in range(P_sim)]
    t0 = time.perf_counter()
    streams = []
    for r in range(P_sim):
        if cfg.get("bucket"):
            i, v, eps[r] = oracle.ef_topk_bucketed(eps[r], grads[r], 0.01, k, cfg["bucket"])
        else:
            i, v, eps[r] = oracle.ef_topk(eps[r], grads[r], 0.01, k)
        streams.append((i, v))
    if P_sim > 1:
        if cfg["algo"] == "rd":
            oracle.ssar_recursive_double(N_s, streams, n_out=1)
        else:
            a = {"ssar_split": oracle.ALGO_SSAR_SPLIT, "dsar": oracle.ALGO_DSAR_SPLIT}[cfg["algo"]]
            oracle.split_allgather(N_s, streams, algo=a, quant_bits=cfg["bits"], n_out=1)
    return time.perf_counter() - t0


def run_reference(args, cfg, P, rank):
    import oracle
    oracle.build()
    if rank != 0:
        return None
    P_sim = P
    N_s = cfg["N"] // 16            # bounded sample: 1/16 of the vector per rank
    for _ in range(args.warmup):
        oracle_step_time(cfg, P_sim, N_s)
    ts = [oracle_step_time(cfg, P_sim, N_s, seed=s) for s in range(args.steps)]
    t = sum(ts) / len(ts)
    value = P_sim * 4 * N_s / t / 1e9
    sample = f"per step: EF top-k of N/16 = {N_s} values on each of {P_sim} simulated ranks + the collective simulation"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": P, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "N": cfg["N"], "density": cfg["density"]},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return line


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
def main():
    args = parse()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    P = world

    import torch
    import torch.distributed as dist
    if P > 1:   # the reference arm is the CPU oracle: it needs no GPU process group
        dist.init_process_group(backend="gloo" if args.impl == "reference" else "cpu:gloo,cuda:nccl")
    if args.impl == "reference":
        run_reference(args, cfg, P, rank)
        if P > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    import __graft_entry__
    __graft_entry__.build()
    from paper_1802_08021_b200 import sparcml as S
    from paper_1802_08021_b200 import synth

    N = cfg["N"]
    bucket = cfg.get("bucket", 0)
    kk, k = step_k(cfg)                 # kk: top-k's k (per bucket if bucketed), k: entries per rank
    if not bucket:
        assert k == synth.k_for_density(N, cfg["density"])
    algo = {"ssar_split": S.SSAR_SPLIT_ALLGATHER, "rd": S.SSAR_RECURSIVE_DOUBLE,
            "dsar": S.DSAR_SPLIT_ALLGATHER}[cfg["algo"]]
    if algo == S.SSAR_RECURSIVE_DOUBLE and (P & (P - 1)) != 0:
        algo = S.SSAR_SPLIT_ALLGATHER
    opts = S.make_opts(algo=algo, quant_bits=cfg["bits"], seed=1, k_sum_hint=P * k)
    alpha = 0.01

    comm = S.Comm(N, k) if P > 1 else _single_comm(S, N, k)
    grad = torch.from_numpy(synth.gaussian_vector(N, seed=0, rank=rank)).to(dev)
    eps = torch.zeros(N, dtype=torch.float32, device=dev)
    ws = S.TopkWorkspace(N, k, dev)
    out = S.new_out(N, dev)
    if algo == S.SSAR_RECURSIVE_DOUBLE and P > 1:
        idx = torch.empty(k, dtype=torch.int32, device=dev)
        val = torch.empty(k, dtype=torch.float32, device=dev)
    else:   # the top-k writes straight into the result's payload slots (in place, include/sparcml.h)
        idx, val = S.payload_views(out, N, k)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    flush_i64 = flush.view(torch.int64)

    def flush_l2():
        # write a buffer 4x the L2, then read it back: the L2 holds none of the
        # step's data and no dirty lines whose write-back the next kernel would pay
        flush.zero_()
        flush_i64.sum()
    stream = torch.cuda.current_stream()

    def topk():
        S.ef_topk(eps, grad, alpha, kk, ws=ws, idx_out=idx, val_out=val, bucket=bucket)

    def allreduce():
        comm.allreduce(idx, val, N, out=out, opts=opts)

    def barrier():
        torch.cuda.synchronize()
        if P > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        flush_l2()
        topk()
        allreduce()
    barrier()
    res = S.read_result(out)
    assert res.header.status == 0 and res.header.k_sum == P * k

    # The step runs as ONE CUDA graph (launch-bound sequence, captured once):
    # the fused EF top-k kernel, then the sparse allreduce.  A second graph of
    # the same step with an external event-record node between the two splits
    # the step into top-k and allreduce time on the device (the event node
    # itself costs a few microseconds, so the headline times the plain graph).
    ev_m = torch.cuda.Event(enable_timing=True, external=True)
    l0 = S.kernel_launches()
    g_step = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_step):
        topk()
        allreduce()
    launches_per_step = S.kernel_launches() - l0
    g_split = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_split):
        topk()
        ev_m.record()
        allreduce()
    for g in (g_step, g_split):
        for _ in range(max(3, args.warmup)):
            flush_l2()
            barrier()
            comm.barrier()
            g.replay()
    barrier()
    res = S.read_result(out)
    assert res.header.status == 0 and res.header.k_sum == P * k

    def timed(g, tops=None):
        ts = []
        for _ in range(args.steps):
            flush_l2()
            barrier()
            comm.barrier()     # device-side alignment of the ranks before the events
            torch.cuda._sleep(HOLD_CYCLES)   # keep the GPU busy while the host enqueues the step
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            b.synchronize()                 # ev_m is re-recorded by the next replay: read it now
            ts.append(a.elapsed_time(b) / 1e3)
            if tops is not None:
                tops.append(a.elapsed_time(ev_m) / 1e3)
        return ts

    # ---------------- timed region (device events per step, L2 flushed between) ----
    barrier()
    with ClockSampler(local_rank) as clk:
        t_steps = timed(g_step)
        barrier()
    launches = launches_per_step * args.steps
    t_step = sum(t_steps) / args.steps
    # split run (same step + the event node), for the top-k / allreduce breakdown
    t_tops = []
    t_split = timed(g_split, t_tops)
    barrier()
    t_topk_kernel = sum(t_tops) / args.steps    # the fused top-k launch (graph start -> event node)
    t_ar = sum(t_split) / args.steps - t_topk_kernel
    # per-kernel breakdown (eager, every kernel bracketed by library events)
    S.profile_reset()
    S.profile_only(None)
    ev2 = []
    for _ in range(args.steps):
        flush_l2()
        barrier()
        comm.barrier()
        torch.cuda._sleep(HOLD_CYCLES)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        S.profile_enable(True)
        a.record(stream)
        topk()
        allreduce()
        b.record(stream)
        S.profile_enable(False)
        ev2.append((a, b))
    barrier()
    t_eager = sum(a.elapsed_time(b) for a, b in ev2) / 1e3 / args.steps
    prof = {name: S.profile_read(name) for name in S.PROFILED_KERNELS}
    prof = {n: v for n, v in prof.items() if v[0] > 0}
    S.profile_reset()
    res = S.read_result(out)
    K = int(res.header.nnz)
    bytes_recv = int(res.header.bytes_recv)

    # max over ranks
    def allmax(x):
        if P == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_step = allmax(t_step)
    t_ar = allmax(t_ar)
    t_topk_kernel = allmax(t_topk_kernel)
    t_eager = allmax(t_eager)
    value = P * 4 * N / t_step / 1e9

    # roofline: the fused EF top-k kernel (the one HBM pass over the gradient)
    hbm_peak, peak_src = load_peaks()
    t_filter = t_topk_kernel
    alg_bytes = 12 * N + 8 * k          # read eps + grad, write eps (+ k candidates) per launch
    achieved = alg_bytes / t_filter / 1e9 if t_filter > 0 else None
    total_prof_ms = sum(v[1] for v in prof.values())
    kname = ("topk_bucketed_kernel<EF> (ef_topk, bucket %d: one HBM pass, radix select per bucket)" % bucket
             if bucket else "topk_fused_kernel<EF> (ef_topk: one HBM pass + candidate select)")
    roofline = {"kernel": kname, "bound": "hbm",
                "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": (achieved / hbm_peak) if achieved else None,
                "traffic": ncu_traffic("topk_bucketed" if bucket else "topk"),
                "alg_bytes_per_launch": alg_bytes, "avg_launch_us": t_filter * 1e6, "peak_source": peak_src,
                # share of the step on the device, from the split graph (its event node sits in the
                # allreduce part, so this under-states the top-k share a little)
                "share_of_step": t_topk_kernel / (t_topk_kernel + t_ar) if t_topk_kernel + t_ar > 0 else None}

    # ---------------- e2e through the C ABI with host buffers ----------------
    e2e = None
    if not args.no_e2e:
        gh = torch.empty(N, dtype=torch.float32, pin_memory=True)
        gh.copy_(grad.cpu())
        hdr_h = torch.empty(64, dtype=torch.uint8, pin_memory=True)
        pay_h = torch.empty(S.result_bytes(N), dtype=torch.uint8, pin_memory=True)
        t_e2e, d2h = 0.0, 0
        for it in range(max(2, args.steps // 2)):
            flush_l2()
            barrier()
            comm.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            grad.copy_(gh, non_blocking=True)                 # H2D of the step's input
            topk()                                            # the public API, eager
            allreduce()
            hdr_h.copy_(out[:64], non_blocking=True)          # D2H: header, then the payload
            stream.synchronize()
            h = S.Header.from_buffer_copy(bytes(hdr_h.numpy()))
            n = int(h.nnz)
            if h.repr == S.REPR_SPARSE:
                pay_h[64:64 + 4 * n].copy_(out[64:64 + 4 * n], non_blocking=True)
                pay_h[h.val_offset:h.val_offset + 4 * n].copy_(out[h.val_offset:h.val_offset + 4 * n],
                                                                non_blocking=True)
                d2h = 64 + 8 * n
            else:
                pay_h[64:64 + 4 * N].copy_(out[64:64 + 4 * N], non_blocking=True)
                d2h = 64 + 4 * N
            b.record(stream)
            stream.synchronize()
            if it > 0:
                t_e2e += a.elapsed_time(b) / 1e3
        t_e2e = allmax(t_e2e / (max(2, args.steps // 2) - 1))
        e2e = {"value": P * 4 * N / t_e2e / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 4 * N,
               "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e * 1e3}

    # ---------------- in-run dense baseline (the paper's baseline) ------
    dense_us = None
    if P > 1:
        buf = torch.randn(N, device=dev)
        for _ in range(3):
            dist.all_reduce(buf)
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(10):
            dist.all_reduce(buf)
        b.record(stream)
        barrier()
        dense_us = allmax(a.elapsed_time(b) / 10 * 1e3)

    # ---------------- CPU oracle baseline (rank 0, N = 1 only) ----------------
    cpu = None
    if rank == 0 and P == 1 and not args.no_cpu:
        import oracle
        oracle.build()
        N_s = N // 4
        ts = [oracle_step_time(cfg, 1, N_s, seed=s) for s in range(2)]
        t_cpu = min(ts)
        cpu = {"value": 4 * N_s / t_cpu / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": f"EF top-k{' (bucketed)' if bucket else ''} (qsort) of N/4 = {N_s} values, 1 rank, best of 2; "
                         f"{t_cpu:.2f} s per sample on one host core"}

    clocks = clk.summary()
    clocks["sm_mhz"] = allmax(clocks["sm_mhz"] or 0.0) if P > 1 else clocks["sm_mhz"]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": P, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "N": N, "k_per_rank": k,
                       "bucket": bucket or None, "k_per_bucket": kk if bucket else None,
                       "density": cfg["density"], "P": P, "algo": {1: "SSAR_Recursive_double",
                       2: "SSAR_Split_allgather", 3: "DSAR_Split_allgather"}[algo],
                       "quant_bits": cfg["bits"], "l2": "flushed before every step (512 MiB write + 512 MiB read, no dirty lines left)",
                       "exchange": "CUDA IPC over NVLink (fused push/pull kernels)" if P > 1 else "none (P=1)"},
            "latency_us": t_step * 1e6, "allreduce_us": t_ar * 1e6, "topk_us": t_topk_kernel * 1e6,
            "timing": "one CUDA graph per step (top-k, allreduce); top-k/allreduce split from a second graph with an external event node between them; eager API step measured too",
            "eager_ms_per_step": t_eager * 1e3,
            "result_nnz": K, "bytes_recv_per_rank": bytes_recv,
            "exchange_gbs_per_rank": bytes_recv / t_ar / 1e9 if P > 1 else None,
            "dense_nccl_allreduce_us": dense_us,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
            "kernel_ms_per_step": {n: v[1] / args.steps for n, v in prof.items()},
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if P > 1:
        dist.barrier()
        comm.close()
        dist.destroy_process_group()


def _single_comm(S, N, k):
    """P = 1: a one-rank world (no process group needed)."""
    class One(S.Comm):
        def __init__(self):
            import ctypes as C
            import torch
            h = C.c_void_p()
            S._check(S._lib.sparcml_comm_create(C.byref(h), 1, 0, torch.cuda.current_device(), N, k))
            self._h, self.P, self.rank, self.device = h, 1, 0, torch.cuda.current_device()
    return One()


if __name__ == "__main__":
    main()
