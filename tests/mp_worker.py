"""torchrun worker for tests/test_multigpu.py: one rank per GPU, CUDA-IPC
world, every algorithm checked against the oracle on every rank."""
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
    if os.environ.get("SPARCML_MP_VERBOSE"):
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ["SPARCML_MP_VERBOSE"]), exit=True)
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    cases = [
        ("rd", 200_003, 3000, S.SSAR_RECURSIVE_DOUBLE, 0),
        ("rd-dense", 50_000, 20_000, S.SSAR_RECURSIVE_DOUBLE, 0),
        ("ssar", 1 << 20, 10_000, S.SSAR_SPLIT_ALLGATHER, 0),
        ("dsar", 1 << 20, 200_000, S.DSAR_SPLIT_ALLGATHER, 0),
        ("dsar4", 1 << 20, 200_000, S.DSAR_SPLIT_ALLGATHER, 4),
        ("auto", 1 << 20, 300_000, S.ALGO_AUTO, 2),
        ("auto-ssar", 1 << 20, 100_000, S.ALGO_AUTO, 0),   # device decides SSAR (both concat variants launched)
        ("ssar-big", 1 << 24, 167_772, S.SSAR_SPLIT_ALLGATHER, 0),
        # fp64 values: the _f64 entry points, oracle's fp64 build
        ("f64-rd", 200_003, 3000, S.SSAR_RECURSIVE_DOUBLE, 0),
        ("f64-ssar", 1 << 20, 10_000, S.SSAR_SPLIT_ALLGATHER, 0),
        ("f64-dsar", 1 << 20, 200_000, S.DSAR_SPLIT_ALLGATHER, 0),
        ("f64-auto", 1 << 20, 300_000, S.ALGO_AUTO, 0),
    ]
    max_N = max(c[1] for c in cases)
    max_k = max(c[2] for c in cases)
    comm = S.Comm(max_N, max_k)
    fails = 0
    for rep in range(2):
        for name, N, k, algo, bits in cases:
            if os.environ.get("SPARCML_MP_VERBOSE"):
                print(f"rank {rank}: rep {rep} case {name}", flush=True)
            f64 = name.startswith("f64")
            dt = np.float64 if f64 else np.float32
            streams = synth.uniform_streams(P, N, k, seed=rep * 10 + len(name), kind="normal64" if f64 else "normal")
            i, v = streams[rank]
            it = torch.from_numpy(i.view(np.int32)).cuda()
            vt = torch.from_numpy(v).cuda()
            opts = S.make_opts(algo=algo, quant_bits=bits, seed=3)
            out = comm.allreduce(it, vt, N, opts=opts)
            res = S.read_result(out)
            if algo == S.SSAR_RECURSIVE_DOUBLE:
                ref, st = oracle.ssar_recursive_double(N, streams, dtype=dt)
            else:
                oa = {S.SSAR_SPLIT_ALLGATHER: oracle.ALGO_SSAR_SPLIT, S.DSAR_SPLIT_ALLGATHER: oracle.ALGO_DSAR_SPLIT,
                      S.ALGO_AUTO: oracle.ALGO_AUTO}[algo]
                ref, st, _ = oracle.split_allgather(N, streams, algo=oa, quant_bits=bits, seed=3, dtype=dt)
            d, ei, ev = ref[rank]
            ok = res.header.status == 0 and res.dense == d and res.header.k_sum == P * k
            if ok and d:
                ok = np.array_equal(res.val.cpu().numpy(), ev)
            elif ok:
                ok = (np.array_equal(res.idx.cpu().numpy().view(np.uint32), ei)
                      and np.array_equal(res.val.cpu().numpy(), ev))
            ok = ok and res.header.bytes_recv == st[rank]["bytes_recv"] and res.header.bytes_sent == st[rank]["bytes_sent"]
            if not ok:
                fails += 1
                print(f"rank {rank}: case {name} rep {rep} MISMATCH (dense {res.dense} vs {d}, "
                      f"nnz {res.header.nnz}, status {res.header.status})", flush=True)
    fails += layerwise(comm, rank, P)
    fails += allgather(comm, rank, P)
    fails += allgather_skewed(comm, rank, P)
    fails += algorithm1(comm, rank, P)
    comm.close()
    fails += failures(rank, P)
    t = torch.tensor([fails])
    dist.all_reduce(t)
    dist.destroy_process_group()
    if rank == 0:
        print(f"multigpu P={P}: {'OK' if t.item() == 0 else 'FAILED'} ({int(t.item())} mismatches)", flush=True)
    sys.exit(0 if t.item() == 0 else 1)


def layerwise(comm, rank, P):
    """NEXT row 1: layer-wise non-blocking allreduces on a communication stream,
    overlapped with top-k work on the compute stream, and the tensor-fused
    variant (one allreduce over all layers), both against the oracle per layer."""
    dims = [100_003, 2_000_000, 777, 500_000]
    ks = [1000, 20_000, 50, 5000]
    off = S.layer_offsets(dims)
    layers = [synth.uniform_streams(P, dims[l], ks[l], seed=40 + l, kind="normal") for l in range(len(dims))]
    mine = [(torch.from_numpy(layers[l][rank][0].view(np.int32)).cuda(), torch.from_numpy(layers[l][rank][1]).cuda())
            for l in range(len(dims))]
    comp, cs = torch.cuda.current_stream(), torch.cuda.Stream()
    x = torch.randn(1 << 22, device="cuda")
    ws = S.TopkWorkspace(x.numel(), 4096)
    opts = S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER)
    reqs = []
    for l in reversed(range(len(dims))):           # backward order, as gradients appear
        S.topk_sparsify(x, 4096, ws=ws)              # compute-stream work to overlap with
        ev = torch.cuda.Event()
        ev.record(comp)
        cs.wait_event(ev)
        reqs.append((l, comm.allreduce_async(mine[l][0], mine[l][1], dims[l], opts=opts, stream=cs)))
    fails = 0
    for l, rq in reqs:
        rq.wait(comp)
        res = rq.result()
        ref, _, _ = oracle.split_allgather(dims[l], layers[l], algo=oracle.ALGO_SSAR_SPLIT)
        wmask, want = oracle.result_to_dense(ref[rank], dims[l])
        got = np.zeros(dims[l], np.float32)
        gmask = np.ones(dims[l], np.uint8)
        if res.dense:
            got[:] = res.val.cpu().numpy()
        else:
            ii = res.idx.cpu().numpy().astype(np.int64)
            got[ii] = res.val.cpu().numpy()
            gmask[:] = 0
            gmask[ii] = 1
        if not (np.array_equal(got, want) and np.array_equal(gmask, wmask)):
            fails += 1
            print(f"rank {rank}: layer-wise layer {l} MISMATCH", flush=True)
    # fused: one allreduce over sum(N_l), split back by index range
    fi, fv = S.fuse_streams(mine, off)
    out = comm.allreduce(fi, fv, off[-1], opts=opts)
    parts = S.split_result(out, off)
    for l in range(len(dims)):
        ref, _, _ = oracle.split_allgather(dims[l], layers[l], algo=oracle.ALGO_SSAR_SPLIT)
        wmask, want = oracle.result_to_dense(ref[rank], dims[l])
        pi, pv = parts[l]
        got = np.zeros(dims[l], np.float32)
        gmask = np.ones(dims[l], np.uint8)
        if pi is None:
            got[:] = pv.cpu().numpy()
        else:
            ii = pi.cpu().numpy().astype(np.int64) - off[l]
            got[ii] = pv.cpu().numpy()
            gmask[:] = 0
            gmask[ii] = 1
        if not (np.array_equal(got, want) and np.array_equal(gmask, wmask)):
            fails += 1
            print(f"rank {rank}: fused layer {l} MISMATCH", flush=True)
    return fails


def allgather(comm, rank, P):
    """§7 SCD sparse allgather over the IPC world: slices owned in shuffled order."""
    fails = 0
    for N, per, dt in [(1 << 20, 100, np.float32), (1 << 16, 30_000, np.float32), (1 << 20, 300, np.float64),
                       (1 << 16, 32_000, np.float64)]:   # sparse, then K > delta (dense); fp32 and fp64
        rng = np.random.default_rng(N + per)
        bounds = np.linspace(0, N, P + 1).astype(np.int64)
        order = rng.permutation(P)
        streams = []
        for r in range(P):
            lo, hi = bounds[order[r]], bounds[order[r] + 1]
            n = min(per, hi - lo)
            i = np.sort(rng.choice(np.arange(lo, hi), n, replace=False)).astype(np.uint32)
            streams.append((i, rng.standard_normal(n).astype(dt)))
        i, v = streams[rank]
        out = comm.allgather(torch.from_numpy(i.view(np.int32)).cuda(), torch.from_numpy(v).cuda(), N)
        g = S.read_result(out)
        ref, st = oracle.sparse_allgather(N, streams, dtype=dt)
        d, ei, ev = ref[rank]
        ok = g.header.status == 0 and g.dense == d
        if ok and d:
            ok = np.array_equal(g.val.cpu().numpy(), ev)
        elif ok:
            ok = np.array_equal(g.idx.cpu().numpy().view(np.uint32), ei) and np.array_equal(g.val.cpu().numpy(), ev)
        ok = ok and g.header.bytes_recv == st[rank]["bytes_recv"]
        if not ok:
            fails += 1
            print(f"rank {rank}: allgather N={N} MISMATCH", flush=True)
    return fails


def allgather_skewed(comm, rank, P):
    """Back-to-back sparse allgathers with no host sync between them while one
    rank runs late (a spin kernel before each of its calls): a fast rank must
    not overwrite a stream the slow one is still pulling (call-parity slots)."""
    N, per, calls = 1 << 18, 4000, 16
    outs, refs = [], []
    for it in range(calls):
        rng = np.random.default_rng(1000 + it)
        bounds = np.linspace(0, N, P + 1).astype(np.int64)
        order = rng.permutation(P)
        streams = []
        for r in range(P):
            lo, hi = bounds[order[r]], bounds[order[r] + 1]
            i = np.sort(rng.choice(np.arange(lo, hi), per, replace=False)).astype(np.uint32)
            streams.append((i, rng.standard_normal(per).astype(np.float32)))
        refs.append(oracle.sparse_allgather(N, streams)[0][rank])
        i, v = streams[rank]
        if rank == P - 1:
            torch.cuda._sleep(200_000)   # ~0.1 ms late for every call
        outs.append(comm.allgather(torch.from_numpy(i.view(np.int32)).cuda(), torch.from_numpy(v).cuda(), N))
    torch.cuda.synchronize()
    fails = 0
    for it in range(calls):
        g = S.read_result(outs[it])
        d, ei, ev = refs[it]
        ok = (g.header.status == 0 and not g.dense and np.array_equal(g.idx.cpu().numpy().view(np.uint32), ei)
              and np.array_equal(g.val.cpu().numpy(), ev))
        if not ok:
            fails += 1
            print(f"rank {rank}: skewed allgather call {it} MISMATCH (status {g.header.status})", flush=True)
    return fails


def failures(rank, P):
    """Failure handling on the IPC world: (1) a rank that skips a collective --
    the others' flag waits give up (header status ERR_TIMEOUT, no hang);
    (2) ranks built with different limits -- connect reports ERR_MISMATCH."""
    fails = 0
    comm = S.Comm(1 << 16, 1000)
    comm.set_timeout(300)
    i, v = synth.uniform_streams(P, 1 << 16, 500, seed=77)[rank]
    if rank != P - 1:   # the last rank is "dead" for this call
        out = comm.allreduce(torch.from_numpy(i.view(np.int32)).cuda(), torch.from_numpy(v).cuda(), 1 << 16,
                             opts=S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER))
        st = S.read_result(out).header.status
        if st != S.ERR_TIMEOUT:
            fails += 1
            print(f"rank {rank}: dead-rank call status {st}, expected ERR_TIMEOUT", flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    comm.close()
    try:
        bad = S.Comm(1 << 16 if rank != 0 else 1 << 17, 1000)
        bad.close()
        fails += 1
        print(f"rank {rank}: mismatched limits were accepted", flush=True)
    except S.SparcmlError as e:
        if e.status != S.ERR_MISMATCH:
            fails += 1
            print(f"rank {rank}: mismatched limits gave status {e.status}, expected ERR_MISMATCH", flush=True)
    dist.barrier()
    return fails


def algorithm1(comm, rank, P):
    """Algorithm 1 through S.algorithm1_step on the IPC world, with
    QSGD on the selected values (R-29), against the step composed from oracle pieces."""
    N, k, alpha, qbits, qb, seed = 300_007, 3000, 0.05, 4, 512, 5
    v = torch.zeros(N, device="cuda")
    e = torch.zeros(N, device="cuda")
    ws = S.TopkWorkspace(N, k)
    vh = np.zeros(N, np.float32)
    eh = [np.zeros(N, np.float32) for _ in range(P)]
    opts = S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER)
    fails = 0
    for step in range(2):
        g = torch.from_numpy(synth.gaussian_vector(N, seed=50 + step, rank=rank)).cuda()
        S.algorithm1_step(comm, v, e, g, alpha, k, q_bits=qbits, q_bucket=qb, q_seed=seed, opts=opts, ws=ws)
        hs = []
        for r in range(P):
            gr = synth.gaussian_vector(N, seed=50 + step, rank=r)
            i, val, eh[r] = oracle.ef_topk(eh[r], gr, alpha, k)
            c, sc = oracle.qsgd_quantize(val, qbits, bucket=qb, seed=seed, ctr_base=r * k)
            hs.append((i, oracle.qsgd_dequantize(c, sc, len(val), qbits, qb)))
        ref, _, _ = oracle.split_allgather(N, hs, algo=oracle.ALGO_SSAR_SPLIT)
        _, gd = oracle.result_to_dense(ref[rank], N)
        vh = (vh - gd).astype(np.float32)
        if not (np.array_equal(v.cpu().numpy(), vh) and np.array_equal(e.cpu().numpy(), eh[rank])):
            fails += 1
            print(f"rank {rank}: algorithm 1 step {step} MISMATCH", flush=True)
    return fails


if __name__ == "__main__":
    main()
