"""Small parity cases for compute-sanitizer runs (memcheck / racecheck /
synccheck, one tool per run): every kernel family at sizes the
sanitizers finish in minutes, each checked against the oracle.

  compute-sanitizer --tool memcheck --error-exitcode 17 python tests/sanitizer_smoke.py

Not collected by pytest (no test_ prefix); profiles/r02_sanitizer_*.log hold
the committed runs.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1802_08021_b200 import sparcml as S, synth  # noqa: E402


def cu_idx(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(name, ok):
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        raise SystemExit(1)


def main():
    oracle.build()
    torch.cuda.set_device(0)
    # merge (merge_span)
    (ia, va), (ib, vb) = synth.uniform_streams(2, 9000, [3000, 5000], seed=1)
    io, vo = S.merge_sum(cu_idx(ia), cu(va), cu_idx(ib), cu(vb))
    eo, ev = oracle.merge_sum(ia, va, ib, vb)
    check("merge_sum", np.array_equal(io.cpu().numpy().view(np.uint32), eo) and np.array_equal(vo.cpu().numpy(), ev))
    # global top-k (sample path, tiny path, EF) with one reused workspace
    ws = S.TopkWorkspace(70_000, 700)
    for N, k, ef in [(70_000, 700, False), (4097, 4096, False), (70_000, 650, True), (1000, 10, True)]:
        x = synth.gaussian_vector(N, seed=N + k)
        if ef:
            g = synth.gaussian_vector(N, seed=N)
            xt = cu(x)
            i, v = S.ef_topk(xt, cu(g), 0.1, k, ws=ws)
            ei, evv, ee = oracle.ef_topk(x, g, 0.1, k)
            ok = np.array_equal(xt.cpu().numpy(), ee)
        else:
            i, v = S.topk_sparsify(cu(x), k, ws=ws)
            ei, evv = oracle.topk(x, k)
            ok = True
        check(f"topk N={N} k={k} ef={ef}", ok and np.array_equal(i.cpu().numpy().view(np.uint32), ei)
              and np.array_equal(v.cpu().numpy(), evv))
    # bucketed top-k
    x = synth.gaussian_vector(5000, seed=3)
    i, v = S.topk_sparsify(cu(x), 7, bucket=512)
    ei, evv = oracle.topk_bucketed(x, 7, 512)
    check("topk bucketed", np.array_equal(i.cpu().numpy().view(np.uint32), ei) and np.array_equal(v.cpu().numpy(), evv))
    # QSGD codec
    x = synth.gaussian_vector(1000, seed=4)
    c, s = S.quantize(cu(x), 4, bucket=256, seed=9, ctr_base=5)
    ec, es = oracle.qsgd_quantize(x, 4, bucket=256, seed=9, ctr_base=5)
    check("qsgd", np.array_equal(c.cpu().numpy(), ec) and np.array_equal(s.cpu().numpy(), es))
    # collectives on a loopback world of 4 ranks
    P, N = 4, 20_000
    streams = synth.uniform_streams(P, N, 600, seed=7)
    w = S.LocalWorld(P, N, 8000)
    dev = [(cu_idx(i), cu(v)) for i, v in streams]
    for name, algo, bits in [("rd", S.SSAR_RECURSIVE_DOUBLE, 0), ("ssar", S.SSAR_SPLIT_ALLGATHER, 0),
                             ("dsar", S.DSAR_SPLIT_ALLGATHER, 0), ("dsar4", S.DSAR_SPLIT_ALLGATHER, 4)]:
        outs = w.allreduce(dev, N, opts=S.make_opts(algo=algo, quant_bits=bits, seed=2))
        if algo == S.SSAR_RECURSIVE_DOUBLE:
            ref, _ = oracle.ssar_recursive_double(N, streams)
        else:
            oa = oracle.ALGO_SSAR_SPLIT if algo == S.SSAR_SPLIT_ALLGATHER else oracle.ALGO_DSAR_SPLIT
            ref, _, _ = oracle.split_allgather(N, streams, algo=oa, quant_bits=bits, seed=2)
        ok = True
        for r in range(P):
            g = S.read_result(outs[r])
            d, ei, evv = ref[r]
            if g.header.status != 0 or g.dense != bool(d):
                ok = False
            elif d:
                ok &= np.array_equal(g.val.cpu().numpy(), evv)
            else:
                ok &= np.array_equal(g.idx.cpu().numpy().view(np.uint32), ei) and np.array_equal(g.val.cpu().numpy(), evv)
        check(f"allreduce {name}", ok)
    # sparse allgather (disjoint ranges)
    part = N // P
    rng = np.random.default_rng(5)
    ag = []
    for r in range(P):
        i = np.sort(rng.choice(part, 300, replace=False)).astype(np.uint32) + np.uint32(r * part)
        ag.append((i, rng.standard_normal(300).astype(np.float32)))
    outs = w.allgather([(cu_idx(i), cu(v)) for i, v in ag], N)
    ref, _ = oracle.sparse_allgather(N, ag)
    ok = all(np.array_equal(S.read_result(outs[r]).idx.cpu().numpy().view(np.uint32), ref[r][1]) for r in range(P))
    check("allgather", ok)
    w.close()
    torch.cuda.synchronize()
    print("sanitizer smoke: all cases ok", flush=True)


if __name__ == "__main__":
    main()
