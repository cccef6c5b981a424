#!/usr/bin/env python
"""bench.py — SparCML hot path on B200 (SURVEY §8(d) measurement protocol).

Workloads (BASELINE.json configs; --config):
  cfg2 (default): N = 2^24 fp32, 1 % per rank: EF top-k of a Gaussian gradient
        (a uniform-random support of exactly k, the paper's micro-benchmark input
        P:937-938) + SSAR_Split_allgather of the P streams.
  cfg3: top-k 0.1 % of a 25,557,032-parameter gradient + recursive doubling.
  cfg4: 10 % per rank, DSAR_Split_allgather with 4-bit QSGD.
  bucket512: the DNN selector, 4 of every 512, + split-allgather.
  cfg1: P = 4 simulated ranks, N = 4096, k = 64, recursive doubling.
  cfg5: logistic-regression gradients (N = 3,231,961, clustered support), AUTO.
cfg1 and cfg5 name their rank count (4, 8); with fewer processes every process
runs that many simulated ranks on its GPU (a loopback world, kernels in rank
order), stated in config.world.

One step = the whole hot path over one batch: EF top-k (where the config has
one) then the sparse allreduce, replayed as one CUDA graph.  Inputs cycle
through 5 dataset seeds (step i uses seed i mod 5; P:943-944 reports p25/p50/
p75 over seeds x reps).  value = whole-job result GB/s = P * result bytes / t
(8K for a sparse result, 4N dense: SURVEY §8(d)); dense_equiv_gbs = P*4N/t.

Timing: W untimed warm-ups, then exactly K steps, each bracketed by CUDA
events on the launching stream after an L2 flush (512 MiB write + read back),
a host barrier, the library's device barrier and a ~0.5 ms spin kernel (the
start event fires when the GPU reaches the step); max over ranks.

Launch: python bench.py [--gpus N --steps K --warmup W --config cfgX]; N > 1
under torchrun (one rank per GPU).  --impl reference times the CPU oracle.
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
NSEEDS = 5

CONFIGS = {
    "cfg1": dict(desc="BASELINE configs[0]: P=4 simulated ranks, N=4096 fp32, k=64 random nonzeros per rank, "
                      "SSAR_Recursive_double", kind="streams", N=4096, k=64, algo="rd", bits=0, sim=4, streams="uniform"),
    "cfg2": dict(desc="BASELINE configs[1]: N=16M (2^24) fp32, density 1% uniform-random support per rank "
                      "(EF top-k of a Gaussian gradient), SSAR_Split_allgather",
                 kind="topk", N=1 << 24, density=0.01, algo="ssar_split", bits=0),
    "cfg3": dict(desc="BASELINE configs[2]: top-k 0.1% of a 25,557,032-parameter Gaussian gradient, "
                      "SSAR_Recursive_double", kind="topk", N=25_557_032, density=0.001, algo="rd", bits=0),
    "cfg4": dict(desc="BASELINE configs[3]: N=2^24, density 10%, DSAR_Split_allgather with QSGD 4-bit",
                 kind="topk", N=1 << 24, density=0.10, algo="dsar", bits=4),
    "cfg5": dict(desc="BASELINE configs[4]: naturally sparse logistic-regression gradients, N=3,231,961 features, "
                      "clustered (Zipf-ranked 256-wide blocks) support, 1000 samples x 100 features per rank, AUTO",
                 kind="streams", N=3_231_961, algo="auto", bits=0, sim=8, streams="lr"),
    "bucket512": dict(desc="NEXT (SURVEY 8f rank 2): bucketed EF top-k, 4 of every 512 (P:1238), of a "
                           "25,557,032-parameter Gaussian gradient, SSAR_Split_allgather",
                      kind="topk", N=25_557_032, density=4 / 512, algo="ssar_split", bits=0, bucket=512, kb=4),
}


def step_k(cfg, N=None):
    """(k passed to top-k, entries it writes)."""
    N = cfg["N"] if N is None else N
    if cfg.get("bucket"):
        B, kb = cfg["bucket"], cfg["kb"]
        full, tail = divmod(N, B)
        return kb, full * min(kb, B) + (min(kb, tail) if tail else 0)
    if "k" in cfg:
        return cfg["k"], cfg["k"]
    k = max(1, int(cfg["density"] * N))
    return k, k


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["sparcml", "reference"], default="sparcml")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the in-run baselines and merge rooflines")
    return ap.parse_args()


HOLD_CYCLES = 1_000_000   # ~0.5 ms spin ahead of each timed step (host enqueue jitter is not kernel time)


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def load_json(rel):
    try:
        with open(os.path.join(ROOT, rel)) as f:
            return json.load(f)
    except Exception:
        return None


def load_peaks():
    d = load_json("MEASURED_PEAKS.json")
    if d and "hbm_gbs" in d:
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def nvlink_peak():
    d = load_json("profiles/nvlink_peak.json")
    if d and d.get("best_pull_gbs"):
        return float(d["best_pull_gbs"]), "measured (profiles/nvlink_peak.json: kernel 16-byte peer loads, best pair)"
    return 770.0, "fallback (B200_PROFILING.md peer copy 770 GB/s per direction)"


def ncu_traffic(kernel: str):
    d = load_json("profiles/ncu_summary.json")
    try:
        return d["kernels"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def pct(xs, q):
    xs = sorted(xs)
    if not xs:
        return None
    i = (len(xs) - 1) * q / 100.0
    lo = int(i)
    hi = min(lo + 1, len(xs) - 1)
    return xs[lo] + (xs[hi] - xs[lo]) * (i - lo)


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
# CPU oracle (reference arm and cpu_baseline): plain single-threaded C
# ---------------------------------------------------------------------------
def oracle_streams(cfg, P_sim, N_s, seed):
    from paper_1802_08021_b200 import synth
    if cfg.get("streams") == "lr":
        return synth.lr_gradient_streams(P_sim, N_s, seed=seed)
    return synth.uniform_streams(P_sim, N_s, step_k(cfg, N_s)[0], seed=seed)


def oracle_step_time(cfg, P_sim, N_s, seed=0):
    """One step of the workload at dimension N_s for P_sim ranks on the CPU
    oracle (EF top-k per rank where the config has one, then the collective
    simulation).  Returns seconds."""
    import numpy as np
    import oracle
    from paper_1802_08021_b200 import synth
    if cfg["kind"] == "topk":
        k, _ = step_k(cfg, N_s)
        grads = [synth.gaussian_vector(N_s, seed=seed, rank=r) for r in range(P_sim)]
        eps = [np.zeros(N_s, np.float32) for _ in range(P_sim)]
    else:
        streams = oracle_streams(cfg, P_sim, N_s, seed)
    t0 = time.perf_counter()
    if cfg["kind"] == "topk":
        streams = []
        for r in range(P_sim):
            if cfg.get("bucket"):
                i, v, eps[r] = oracle.ef_topk_bucketed(eps[r], grads[r], 0.01, k, cfg["bucket"])
            else:
                i, v, eps[r] = oracle.ef_topk(eps[r], grads[r], 0.01, k)
            streams.append((i, v))
    if P_sim > 1:
        if cfg["algo"] == "rd" and (P_sim & (P_sim - 1)) == 0:
            res, _ = oracle.ssar_recursive_double(N_s, streams, n_out=1)
        else:
            a = {"ssar_split": oracle.ALGO_SSAR_SPLIT, "dsar": oracle.ALGO_DSAR_SPLIT, "auto": oracle.ALGO_AUTO,
                 "rd": oracle.ALGO_SSAR_SPLIT}[cfg["algo"]]
            res = oracle.split_allgather(N_s, streams, algo=a, quant_bits=cfg["bits"], n_out=1)[0]
        d, i, _ = res[0]
    else:
        d, i = False, streams[0][0]
    t = time.perf_counter() - t0
    return t, (4 * N_s if d else 8 * len(i))


def oracle_sample(cfg, P):
    """The bounded sample the CPU legs time: full N on one simulated rank at
    P = 1 (~2-3 s of single-core work per step for the top-k configs), 1/P of
    N per rank for P simulated ranks otherwise (the same CPU work per step)."""
    P_sim = max(P, cfg.get("sim", 1))
    frac = 1 if P_sim == 1 or cfg["kind"] == "streams" else P_sim
    return P_sim, cfg["N"] // frac


def run_reference(args, cfg, P, rank):
    import oracle
    oracle.build()
    if rank != 0:
        return None
    P_sim, N_s = oracle_sample(cfg, P)
    for s in range(args.warmup):
        oracle_step_time(cfg, P_sim, N_s, seed=s % NSEEDS)
    runs = [oracle_step_time(cfg, P_sim, N_s, seed=s % NSEEDS) for s in range(args.steps)]
    ts = [r[0] for r in runs]
    t = sum(ts) / len(ts)
    value = P * statistics.mean(r[1] for r in runs) / t / 1e9   # result GB/s, the GPU arm's definition
    sample = (f"per step: {'EF top-k of ' + str(N_s) + ' values on each of ' if cfg['kind'] == 'topk' else ''}"
              f"{P_sim} simulated rank(s) + the collective simulation (N = {N_s}"
              f"{'' if N_s == cfg['N'] else ', 1/' + str(cfg['N'] // N_s) + ' of the workload N'})")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": P, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "N": cfg["N"]},
            "latency_us": {"p25": pct(ts, 25) * 1e6, "p50": pct(ts, 50) * 1e6, "p75": pct(ts, 75) * 1e6},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
            "host": host_info(),
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
    B = Bench(args, cfg, P, rank, local_rank, dev, torch, dist, S)
    line = B.run()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if P > 1:
        dist.barrier()
        B.close()
        dist.destroy_process_group()


class Bench:
    def __init__(self, args, cfg, P, rank, local_rank, dev, torch, dist, S):
        self.args, self.cfg, self.P, self.rank, self.local_rank = args, cfg, P, rank, local_rank
        self.dev, self.torch, self.dist, self.S = dev, torch, dist, S
        self.N = cfg["N"]
        self.flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        self.stream = torch.cuda.current_stream()

    # ---- plumbing ---------------------------------------------------------
    def flush_l2(self):
        # write a buffer 4x the L2, then read it back: the L2 holds none of the
        # step's data and no dirty lines whose write-back the next kernel would pay
        self.flush_buf.zero_()
        self.flush_buf.view(self.torch.int64).sum()

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.P > 1:
            self.dist.barrier()

    def allmax(self, x):
        if self.P == 1 or x is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def timed(self, fn, steps, comm=None, pre=None):
        """Per-step device time (s) of fn(i) for i in range(steps), L2 flushed before each."""
        torch = self.torch
        ts = []
        for i in range(steps):
            if pre:
                pre(i)
            self.flush_l2()
            self.barrier()
            if comm is not None:
                comm.barrier()
            torch.cuda._sleep(HOLD_CYCLES)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
            fn(i)
            b.record(self.stream)
            b.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        return ts

    def close(self):
        if getattr(self, "comm", None) is not None:
            self.comm.close()

    # ---- the workload -----------------------------------------------------
    def run(self):
        if self.cfg["kind"] == "topk":
            return self.run_topk()
        return self.run_streams()

    def algo_id(self, P_world):
        S, a = self.S, self.cfg["algo"]
        algo = {"ssar_split": S.SSAR_SPLIT_ALLGATHER, "rd": S.SSAR_RECURSIVE_DOUBLE,
                "dsar": S.DSAR_SPLIT_ALLGATHER, "auto": S.ALGO_AUTO}[a]
        if algo == S.SSAR_RECURSIVE_DOUBLE and (P_world & (P_world - 1)) != 0:
            algo = S.SSAR_SPLIT_ALLGATHER
        return algo

    def make_comm(self, N, k):
        S = self.S
        if self.P > 1:
            return S.Comm(N, k)

        class One(S.Comm):
            def __init__(self):
                import ctypes as C
                import torch
                h = C.c_void_p()
                S._check(S._lib.sparcml_comm_create(C.byref(h), 1, 0, torch.cuda.current_device(), N, k))
                self._h, self.P, self.rank, self.device = h, 1, 0, torch.cuda.current_device()
        return One()

    def run_topk(self):
        torch, S, cfg, P, N = self.torch, self.S, self.cfg, self.P, self.N
        from paper_1802_08021_b200 import synth
        bucket = cfg.get("bucket", 0)
        kk, k = step_k(cfg)
        algo = self.algo_id(P)
        opts = S.make_opts(algo=algo, quant_bits=cfg["bits"], seed=1, k_sum_hint=P * k)
        alpha = 0.01
        self.comm = comm = self.make_comm(N, k)
        grads = [torch.from_numpy(synth.gaussian_vector(N, seed=s, rank=self.rank)).to(self.dev) for s in range(NSEEDS)]
        eps = torch.zeros(N, dtype=torch.float32, device=self.dev)
        ws = S.TopkWorkspace(N, k, self.dev)
        out = S.new_out(N, self.dev)
        if algo == S.SSAR_RECURSIVE_DOUBLE and P > 1:
            idx = torch.empty(k, dtype=torch.int32, device=self.dev)
            val = torch.empty(k, dtype=torch.float32, device=self.dev)
        else:   # the top-k writes straight into the result's payload slots (in place, include/sparcml.h)
            idx, val = S.payload_views(out, N, k)

        def topk(s):
            S.ef_topk(eps, grads[s], alpha, kk, ws=ws, idx_out=idx, val_out=val, bucket=bucket)

        def allreduce():
            comm.allreduce(idx, val, N, out=out, opts=opts)

        for i in range(max(3, self.args.warmup)):
            self.flush_l2()
            topk(i % NSEEDS)
            allreduce()
        self.barrier()
        res = S.read_result(out)
        assert res.header.status == 0 and res.header.k_sum == P * k, (res.header.status, res.header.k_sum)

        # one CUDA graph per seed: the EF top-k kernel, then the allreduce's launches;
        # a second graph of seed 0 with an external event-record node between the two
        # splits the step into top-k and allreduce time
        ev_m = torch.cuda.Event(enable_timing=True, external=True)
        l0 = S.kernel_launches()
        graphs = []
        for s in range(NSEEDS):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                topk(s)
                allreduce()
            graphs.append(g)
        launches_per_step = (S.kernel_launches() - l0) // NSEEDS
        g_split = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_split):
            topk(0)
            ev_m.record()
            allreduce()
        for g in graphs + [g_split]:
            for _ in range(max(3, self.args.warmup)):
                self.flush_l2()
                self.barrier()
                comm.barrier()
                g.replay()
        self.barrier()
        assert S.read_result(out).header.status == 0

        # ---------------- timed region ----------------
        K = self.args.steps
        self.barrier()
        with ClockSampler(self.local_rank) as clk:
            t_steps = self.timed(lambda i: graphs[i % NSEEDS].replay(), K, comm)
            self.barrier()
        res = S.read_result(out)
        K_res, dense_res = int(res.header.nnz), res.header.repr == S.REPR_DENSE
        bytes_recv = int(res.header.bytes_recv)
        # split run (seed 0's graph with the event node) for the top-k / allreduce breakdown
        t_top_list, t_ar_list = [], []
        for i in range(max(5, K // 5)):
            self.flush_l2()
            self.barrier()
            comm.barrier()
            torch.cuda._sleep(HOLD_CYCLES)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
            g_split.replay()
            b.record(self.stream)
            b.synchronize()
            t_top_list.append(a.elapsed_time(ev_m) / 1e3)
            t_ar_list.append(ev_m.elapsed_time(b) / 1e3)
        t_topk = self.allmax(statistics.mean(t_top_list))
        t_ar = self.allmax(statistics.mean(t_ar_list))
        # the top-k kernel's own launch duration: CUDA events on its stream around each launch
        # (eager, L2 flushed before each; the roofline's denominator)
        t_topk_launch = self.allmax(statistics.mean(self.timed(lambda i: topk(i % NSEEDS), max(5, K // 5), comm)))
        # per-kernel breakdown (eager, every kernel bracketed by library events)
        S.profile_reset()
        S.profile_only(None)
        for i in range(max(5, K // 5)):
            self.flush_l2()
            self.barrier()
            comm.barrier()
            S.profile_enable(True)
            topk(i % NSEEDS)
            allreduce()
            S.profile_enable(False)
        self.barrier()
        prof = {name: S.profile_read(name) for name in S.PROFILED_KERNELS}
        prof = {n: v for n, v in prof.items() if v[0] > 0}
        nrep = max(5, K // 5)
        S.profile_reset()

        t_mean = self.allmax(statistics.mean(t_steps))
        t_all = t_steps   # rank-local list for percentiles; the mean is max over ranks
        result_bytes = 4 * N if dense_res else 8 * K_res
        hbm_peak, peak_src = load_peaks()
        alg_bytes = 12 * N + 8 * k          # read eps + grad, write eps, k pairs out
        achieved = alg_bytes / t_topk_launch / 1e9
        kname = ("topk_bucketed_kernel<EF> (ef_topk, bucket %d: one HBM pass, radix select per bucket)" % bucket
                 if bucket else "topk_stream_kernel<EF> (ef_topk: TMA-ring streaming pass + candidate select)")
        roofline = {"kernel": kname, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved / hbm_peak, "traffic": ncu_traffic("topk_bucketed" if bucket else "topk"),
                    "alg_bytes_per_launch": alg_bytes, "avg_launch_us": t_topk_launch * 1e6, "peak_source": peak_src,
                    "share_of_step": t_topk / (t_topk + t_ar) if t_topk + t_ar > 0 else None,
                    "timing": "CUDA events on the launching stream around each top-k launch (L2 flushed before "
                              "each), mean, max over ranks; the split graph's top-k segment is topk_us",
                    "graph_segment_us": t_topk * 1e6}
        line = self.common_line(t_mean, t_all, result_bytes, K_res, dense_res, bytes_recv, t_ar, clk, launches_per_step)
        line.update({"topk_us": t_topk * 1e6, "allreduce_us": t_ar * 1e6, "roofline": roofline,
                     "kernel_ms_per_step": {n: v[1] / nrep for n, v in prof.items()},
                     "config": self.config_dict(k, kk, bucket, algo)})
        # ---------------- extras: in-run baselines and merge rooflines ----------------
        if not self.args.no_extra:
            line["baselines"] = self.extra(lambda: self.baselines(grads[0], k, out_k=k, idx=idx, val=val))
            if P == 1:
                line["merge_roofline"] = self.extra(lambda: self.merge_roofline(hbm_peak, peak_src))
                line["owner_roofline"] = self.extra(lambda: self.owner_roofline(hbm_peak, peak_src))
        line["e2e"] = None if self.args.no_e2e else self.e2e_topk(grads[0], topk, allreduce, out)
        line["cpu_baseline"] = self.cpu_baseline()
        return line

    def run_streams(self):
        """cfg1 / cfg5: the allreduce of given per-rank streams (no top-k)."""
        torch, S, cfg, P, N = self.torch, self.S, self.cfg, self.P, self.N
        from paper_1802_08021_b200 import synth
        sim = cfg.get("sim", 1)
        loop = P < sim               # simulate the config's rank count on this GPU
        Pw = sim if loop else P      # ranks of the world the collective runs on
        ranks = list(range(Pw)) if loop else [self.rank]
        per_seed = []
        kmax = 0
        for s in range(NSEEDS):
            if cfg["streams"] == "lr":
                st = synth.lr_gradient_streams(Pw, N, seed=s)
            else:
                st = synth.uniform_streams(Pw, N, cfg["k"], seed=s)
            kmax = max(kmax, max(len(st[r][0]) for r in range(Pw)))
            per_seed.append([(torch.from_numpy(st[r][0].view("int32")).to(self.dev), torch.from_numpy(st[r][1]).to(self.dev))
                             for r in ranks])
        kmax = max(1, kmax)
        algo = self.algo_id(Pw)
        opts = S.make_opts(algo=algo, quant_bits=cfg["bits"])
        if loop:
            self.comm = None
            world = S.LocalWorld(Pw, N, kmax)
            outs = [S.new_out(N, self.dev) for _ in range(Pw)]

            def step(i):
                world.allreduce(per_seed[i % NSEEDS], N, outs=outs, opts=opts)
            comm = None
            out = outs[0]
        else:
            self.comm = comm = self.make_comm(N, kmax)
            out = S.new_out(N, self.dev)

            def step(i):
                idx, val = per_seed[i % NSEEDS][0]
                comm.allreduce(idx, val, N, out=out, opts=opts)
        for i in range(max(3, self.args.warmup)):
            step(i)
        self.barrier()
        assert S.read_result(out).header.status == 0
        graphs = []
        l0 = S.kernel_launches()
        for s in range(NSEEDS):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step(s)
            graphs.append(g)
        launches_per_step = (S.kernel_launches() - l0) // NSEEDS
        for g in graphs:
            for _ in range(3):
                self.barrier()
                if comm is not None:
                    comm.barrier()
                g.replay()
        self.barrier()
        K = self.args.steps
        with ClockSampler(self.local_rank) as clk:
            t_steps = self.timed(lambda i: graphs[i % NSEEDS].replay(), K, comm)
            self.barrier()
        res = S.read_result(out)
        K_res, dense_res = int(res.header.nnz), res.header.repr == S.REPR_DENSE
        t_mean = self.allmax(statistics.mean(t_steps))
        result_bytes = 4 * N if dense_res else 8 * K_res
        line = self.common_line(t_mean, t_steps, result_bytes, K_res, dense_res, int(res.header.bytes_recv),
                                t_mean, clk, launches_per_step, sim_ranks=Pw if loop else None)
        line["allreduce_us"] = t_mean * 1e6
        line["config"] = {"workload": self.args.config, "desc": cfg["desc"], "N": N, "k_per_rank_max": kmax,
                          "P": P, "world": (f"loopback: {Pw} simulated ranks on each GPU (kernels in rank order)"
                                            if loop else f"{P} ranks, CUDA IPC over NVLink"),
                          "algo": {0: "AUTO", 1: "SSAR_Recursive_double", 2: "SSAR_Split_allgather",
                                   3: "DSAR_Split_allgather"}[algo],
                          "seeds": NSEEDS, "l2": "flushed before every step (512 MiB write + read back)"}
        line["roofline"] = None
        line["e2e"] = None
        if not self.args.no_e2e and not loop:
            line["e2e"] = self.e2e_streams(per_seed[0][0], opts, comm, out)
        line["cpu_baseline"] = self.cpu_baseline()
        if loop:
            world.close()
        return line

    # ---- pieces of the JSON line ------------------------------------------
    def config_dict(self, k, kk, bucket, algo):
        cfg = self.cfg
        return {"workload": self.args.config, "desc": cfg["desc"], "N": self.N, "k_per_rank": k,
                "bucket": bucket or None, "k_per_bucket": kk if bucket else None,
                "density": cfg.get("density"), "P": self.P,
                "algo": {1: "SSAR_Recursive_double", 2: "SSAR_Split_allgather", 3: "DSAR_Split_allgather"}[algo],
                "quant_bits": cfg["bits"], "seeds": NSEEDS,
                "l2": "flushed before every step (512 MiB write + 512 MiB read, no dirty lines left)",
                "exchange": "CUDA IPC over NVLink (fused push/pull kernels)" if self.P > 1 else "none (P=1)"}

    def common_line(self, t_mean, t_all, result_bytes, K_res, dense_res, bytes_recv, t_ar, clk, launches_per_step,
                    sim_ranks=None):
        P, N, K = self.P, self.N, self.args.steps
        seeds = {}
        for i, t in enumerate(t_all):
            seeds.setdefault(i % NSEEDS, []).append(t)
        lat = {"mean": t_mean * 1e6, "p25": pct(t_all, 25) * 1e6, "p50": pct(t_all, 50) * 1e6,
               "p75": pct(t_all, 75) * 1e6,
               "per_seed_p50": [pct(seeds[s], 50) * 1e6 for s in sorted(seeds)],
               "protocol": f"{NSEEDS} dataset seeds x {K // NSEEDS} reps (step i uses seed i mod {NSEEDS}); "
                           "p25/p50/p75 of rank 0's step times, mean = max over ranks (P:943-944)"}
        clocks = clk.summary()
        clocks["sm_mhz"] = self.allmax(clocks["sm_mhz"] or 0.0) if P > 1 else clocks["sm_mhz"]
        nvl, nvl_src = nvlink_peak()
        exch = None
        if P > 1:
            gbs = bytes_recv / t_ar / 1e9
            exch = {"bytes_recv_per_rank": bytes_recv, "allreduce_us": t_ar * 1e6, "gbs_per_rank": gbs,
                    "nvlink_peak_gbs": nvl, "peak_source": nvl_src, "frac": gbs / nvl,
                    "note": "received payload bytes per rank (header.bytes_recv, SURVEY 8(d)) / the allreduce "
                            "segment of the step; the segment includes the merges, so this is a lower bound"}
        return {
            "metric": METRIC, "value": P * result_bytes / t_mean / 1e9, "unit": "GB/s", "n_gpus": P,
            "steps": K, "warmup": self.args.warmup, "ms_per_step": t_mean * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "value_definition": "whole-job result GB/s = P x result bytes / step time (8K sparse, 4N dense; "
                                "SURVEY 8(d)); dense_equiv_gbs = P x 4N / step time",
            "latency_us": lat, "result_nnz": K_res, "result_dense": bool(dense_res),
            "result_gbs_per_rank": result_bytes / t_mean / 1e9, "dense_equiv_gbs": P * 4 * N / t_mean / 1e9,
            "exchange": exch, "gpu_launches": launches_per_step * K, "gpu_launches_per_step": launches_per_step,
            "clocks": clocks, "host": host_info(),
            **({"simulated_ranks": sim_ranks} if sim_ranks else {}),
        }

    def baselines(self, grad, k, out_k, idx, val):
        """In-run library baselines on this box: torch.topk of |acc| (P = 1), the dense NCCL allreduce
        of N fp32 (the paper's baseline) and a naive sparse allgather of the unmerged (idx, val)
        streams (NCCL all_gather, no merge) for P > 1."""
        torch, P, N = self.torch, self.P, self.N
        out = {}
        if P == 1:
            acc = (grad * 0.01).abs()
            ts = self.timed(lambda i: torch.topk(acc, k, sorted=False), 5)
            out["torch_topk_us"] = statistics.mean(ts) * 1e6
            out["torch_topk_note"] = "torch.topk(|acc|, k, sorted=False) alone (no EF update, unsorted indices)"
        if P > 1:
            dist = self.dist
            buf = torch.randn(N, device=self.dev)
            ts = self.timed(lambda i: dist.all_reduce(buf), 5)
            out["dense_nccl_allreduce_us"] = self.allmax(statistics.mean(ts)) * 1e6
            pairs = torch.empty(2 * out_k, dtype=torch.int32, device=self.dev)
            pairs[:out_k] = idx[:out_k]
            pairs[out_k:] = val[:out_k].view(torch.int32)
            gathered = torch.empty(P * 2 * out_k, dtype=torch.int32, device=self.dev)
            ts = self.timed(lambda i: dist.all_gather_into_tensor(gathered, pairs), 5)
            out["naive_sparse_allgather_us"] = self.allmax(statistics.mean(ts)) * 1e6
            out["naive_note"] = "NCCL all_gather of every rank's unmerged k pairs (exchange only, no merge)"
        return out

    @staticmethod
    def extra(fn):
        """An optional extra measurement: a failure is reported in the line, never fatal to it."""
        try:
            return fn()
        except Exception as e:   # noqa: BLE001
            return {"error": f"{type(e).__name__}: {e}"}

    def merge_roofline(self, hbm_peak, peak_src):
        """The union-merge-with-sum (§5.1) at config 4's sizes: two uniform streams of
        k = 10% of 2^24 each (the recursive-doubling stage merge, merge_tile), stand-alone."""
        import ctypes as C
        torch, S = self.torch, self.S
        from paper_1802_08021_b200 import synth
        N = 1 << 24
        k = synth.k_for_density(N, 0.10)
        (ia, va), (ib, vb) = synth.uniform_streams(2, N, k, seed=7)
        cu = lambda a: torch.from_numpy(a).to(self.dev)
        ia, va, ib, vb = cu(ia.view("int32")), cu(va), cu(ib.view("int32")), cu(vb)
        io = torch.empty(2 * k, dtype=torch.int32, device=self.dev)
        vo = torch.empty(2 * k, dtype=torch.float32, device=self.dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=self.dev)
        wsb = int(S._lib.sparcml_ops_workspace_bytes(2 * k))
        ws = torch.zeros(wsb, dtype=torch.uint8, device=self.dev)

        def run(i):
            S._check(S._lib.sparcml_merge_sum(ia.data_ptr(), va.data_ptr(), k, ib.data_ptr(), vb.data_ptr(), k,
                                              io.data_ptr(), vo.data_ptr(), cnt.data_ptr(), ws.data_ptr(), wsb,
                                              S._stream(None)))
        for i in range(3):
            run(i)
        ts = self.timed(run, 10)
        n_out = int(cnt.item())
        t = statistics.mean(ts)
        alg = 8 * (2 * k) + 8 * n_out
        return {"kernel": "merge_jobs_kernel (merge_tile: merge path + warp look-back; the RD stage merge)",
                "bound": "hbm", "work": f"2 x {k} pairs -> {n_out} pairs (N = 2^24, 10% each)",
                "alg_bytes_per_launch": alg, "avg_launch_us": t * 1e6, "achieved": alg / t / 1e9,
                "peak": hbm_peak, "unit": "GB/s", "frac": alg / t / 1e9 / hbm_peak, "peak_source": peak_src}

    def owner_roofline(self, hbm_peak, peak_src):
        """The split-allgather owner's P-way merge (a5) at config 2's sizes, on a loopback world of 4
        simulated ranks (per-launch time from the library's event bracket)."""
        torch, S = self.torch, self.S
        from paper_1802_08021_b200 import synth
        Pw, N = 4, 1 << 24
        k = synth.k_for_density(N, 0.01)
        st = synth.uniform_streams(Pw, N, k, seed=11)
        streams = [(torch.from_numpy(i.view("int32")).to(self.dev), torch.from_numpy(v).to(self.dev)) for i, v in st]
        w = S.LocalWorld(Pw, N, k)
        outs = [S.new_out(N, self.dev) for _ in range(Pw)]
        opts = S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER)
        # the three-kernel split path (push, owner, concat): SSAR known on the host otherwise
        # runs the fused kernel, which has no separate owner launch (read per call)
        fused_env = os.environ.get("SPARCML_FUSED")
        os.environ["SPARCML_FUSED"] = "0"
        for _ in range(3):
            w.allreduce(streams, N, outs=outs, opts=opts)
        self.barrier()
        S.profile_reset()
        S.profile_only("owner")
        for i in range(5):
            self.flush_l2()
            self.barrier()
            S.profile_enable(True)
            w.allreduce(streams, N, outs=outs, opts=opts)
            S.profile_enable(False)
        self.barrier()
        n, ms = S.profile_read("owner")
        S.profile_only(None)
        S.profile_reset()
        if fused_env is None:
            os.environ.pop("SPARCML_FUSED", None)
        else:
            os.environ["SPARCML_FUSED"] = fused_env
        K = int(S.read_result(outs[0]).header.nnz)
        w.close()
        if n == 0:
            return {"kernel": "owner_merge_kernel<4>", "unavailable": "no owner launch was profiled"}
        t = ms / 1e3 / n
        alg = 8 * (Pw * k + K) / Pw   # per owner: its slices of every rank in, its partition result out
        return {"kernel": "owner_merge_kernel<4> (canonical-tree P-way merge in shared memory)", "bound": "hbm",
                "work": f"{Pw} slices of ~{k // Pw} pairs -> ~{K // Pw} pairs per owner (cfg2, loopback P=4)",
                "alg_bytes_per_launch": alg, "avg_launch_us": t * 1e6, "achieved": alg / t / 1e9,
                "peak": hbm_peak, "unit": "GB/s", "frac": alg / t / 1e9 / hbm_peak, "peak_source": peak_src,
                "note": "latency-bound at this size (~2.7 MB per launch): the fraction is reported, not a target"}

    def e2e_topk(self, grad, topk, allreduce, out):
        torch, S, N, P = self.torch, self.S, self.N, self.P
        gh = torch.empty(N, dtype=torch.float32, pin_memory=True)
        gh.copy_(grad.cpu())
        hdr_h = torch.empty(64, dtype=torch.uint8, pin_memory=True)
        pay_h = torch.empty(S.result_bytes(N), dtype=torch.uint8, pin_memory=True)
        t_e2e, d2h = 0.0, 0
        reps = max(3, self.args.steps // 10)
        for it in range(reps):
            self.flush_l2()
            self.barrier()
            if getattr(self, "comm", None) is not None:
                self.comm.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
            grad.copy_(gh, non_blocking=True)                 # H2D of the step's input
            topk(0)                                           # the public API, eager
            allreduce()
            hdr_h.copy_(out[:64], non_blocking=True)          # D2H: header, then the payload
            self.stream.synchronize()
            h = S.Header.from_buffer_copy(bytes(hdr_h.numpy()))
            n = int(h.nnz)
            if h.repr == S.REPR_SPARSE:
                pay_h[64:64 + 4 * n].copy_(out[64:64 + 4 * n], non_blocking=True)
                pay_h[h.val_offset:h.val_offset + 4 * n].copy_(out[h.val_offset:h.val_offset + 4 * n],
                                                                non_blocking=True)
                d2h = 64 + 8 * n
                rb = 8 * n
            else:
                pay_h[64:64 + 4 * N].copy_(out[64:64 + 4 * N], non_blocking=True)
                d2h = 64 + 4 * N
                rb = 4 * N
            b.record(self.stream)
            self.stream.synchronize()
            if it > 0:
                t_e2e += a.elapsed_time(b) / 1e3
        t_e2e = self.allmax(t_e2e / (reps - 1))
        return {"value": P * rb / t_e2e / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 4 * N, "d2h_bytes_per_step": d2h,
                "ms_per_step": t_e2e * 1e3, "dense_equiv_gbs": P * 4 * N / t_e2e / 1e9}

    def e2e_streams(self, st0, opts, comm, out):
        torch, S, N, P = self.torch, self.S, self.N, self.P
        idx_h = st0[0].cpu().pin_memory()
        val_h = st0[1].cpu().pin_memory()
        reps = max(3, self.args.steps // 10)
        t = 0.0
        for it in range(reps):
            self.barrier()
            comm.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
            h, _ = comm.allreduce_host(idx_h, val_h, N, opts=opts)
            b.record(self.stream)
            self.stream.synchronize()
            if it > 0:
                t += a.elapsed_time(b) / 1e3
        t = self.allmax(t / (reps - 1))
        rb = 4 * N if h.repr == S.REPR_DENSE else 8 * int(h.nnz)
        return {"value": P * rb / t / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 8 * idx_h.numel(),
                "d2h_bytes_per_step": S.result_bytes(N), "ms_per_step": t * 1e3}

    def cpu_baseline(self):
        if self.rank != 0 or self.P != 1 or self.args.no_cpu:
            return None
        import oracle
        oracle.build()
        cfg = self.cfg
        P_sim, N_s = oracle_sample(cfg, 1)
        runs = [oracle_step_time(cfg, P_sim, N_s, seed=s) for s in range(3)]
        t, rb = min(runs)
        value = rb / t / 1e9
        sample = (f"{'EF top-k (qsort) of ' + str(N_s) + ' values' if cfg['kind'] == 'topk' else 'the allreduce'} on "
                  f"{P_sim} simulated rank(s)" + ("" if P_sim == 1 else " + the collective simulation") +
                  f", best of 3; {t:.2f} s per step on one host core")
        return {"value": value, "unit": "GB/s (result bytes / s)", "ms_per_step": t * 1e3, "cores": 1,
                "kind": "oracle", "sample": sample, "host": host_info()}


if __name__ == "__main__":
    main()
