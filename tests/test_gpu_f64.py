"""GPU parity of the fp64-value sparse allreduce (values "single or double
precision", §5.1) against the oracle's fp64 build.

Same contract as test_gpu_allreduce.py, with double values: every combine is
one fp64 rounding in the canonical tree order (R-8), so values are compared
bit-exact; a pair is 12 bytes, so delta = floor(N*8/12) and the
header's byte counts follow the oracle's 12/8-byte wire sizes."""
import numpy as np
import pytest

from paper_1802_08021_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1802_08021_b200 import sparcml as S  # noqa: E402

F64 = np.float64
ALGOS = {"rd": S.SSAR_RECURSIVE_DOUBLE, "ssar": S.SSAR_SPLIT_ALLGATHER, "dsar": S.DSAR_SPLIT_ALLGATHER,
         "auto": S.ALGO_AUTO}


def to_cuda(streams):
    return [(torch.from_numpy(np.ascontiguousarray(i, np.uint32).view(np.int32)).cuda(),
             torch.from_numpy(np.ascontiguousarray(v, F64)).cuda()) for i, v in streams]


def oracle_run(orc, N, streams, algo, P):
    if algo == S.SSAR_RECURSIVE_DOUBLE and P > 1:
        res, st = orc.ssar_recursive_double(N, streams, dtype=F64)
        return res, st
    # AUTO runs split-allgather at every size (the crossover measured on the box, csrc/api.cu kRdMaxBytes)
    oalgo = {S.SSAR_SPLIT_ALLGATHER: orc.ALGO_SSAR_SPLIT, S.DSAR_SPLIT_ALLGATHER: orc.ALGO_DSAR_SPLIT,
             S.ALGO_AUTO: orc.ALGO_AUTO, S.SSAR_RECURSIVE_DOUBLE: orc.ALGO_AUTO}[algo]
    res, st, _ = orc.split_allgather(N, streams, algo=oalgo, dtype=F64)
    return res, st


def check(orc, P, N, streams, algo, op=S.OP_SUM, world=None):
    w = world or S.LocalWorld(P, N, max(1, max(len(s[0]) for s in streams)))
    outs = w.allreduce(to_cuda(streams), N, opts=S.make_opts(algo=algo), op=op)
    torch.cuda.synchronize()
    with orc.op_scope(op):
        res, st = oracle_run(orc, N, streams, algo, P)
    for r in range(P):
        g = S.read_result(outs[r])
        d, ei, ev = res[r]
        assert g.header.magic == S.HEADER_MAGIC_F64
        assert g.header.status == 0
        assert g.val.dtype == torch.float64
        assert g.dense == bool(d), f"rank {r}: representation differs"
        if d:
            np.testing.assert_array_equal(g.val.cpu().numpy(), ev)
        else:
            assert g.header.nnz == len(ei)
            np.testing.assert_array_equal(g.idx.cpu().numpy().view(np.uint32), ei)
            np.testing.assert_array_equal(g.val.cpu().numpy(), ev)
        if P > 1:
            assert g.header.bytes_sent == st[r]["bytes_sent"], f"rank {r} bytes_sent"
            assert g.header.bytes_recv == st[r]["bytes_recv"], f"rank {r} bytes_recv"
    return outs


@pytest.mark.parametrize("algo", list(ALGOS))
@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8, 16])
@pytest.mark.parametrize("d", [0.002, 0.05, 0.3])
def test_f64_parity(orc, algo, P, d):
    N = 60_013   # ragged: several merge tiles and windows, last partition longer
    k = max(1, int(d * N))
    streams = synth.uniform_streams(P, N, k, seed=int(d * 1000) + 7 * P, kind="normal64")
    check(orc, P, N, streams, ALGOS[algo])


@pytest.mark.parametrize("op", [S.OP_MAX, S.OP_MIN])
@pytest.mark.parametrize("algo", ["rd", "ssar", "dsar"])
@pytest.mark.parametrize("P", [2, 4, 7])
def test_f64_max_min(orc, op, algo, P):
    N = 40_000
    streams = synth.uniform_streams(P, N, 3000, seed=11 * P + op, kind="normal64")
    check(orc, P, N, streams, ALGOS[algo], op=op)


@pytest.mark.parametrize("P", [2, 4])
def test_f64_switch_at_two_thirds(orc, P):
    # K between N/2 and 2N/3: sparse with double values (fp32 would be dense)
    N = 3000
    streams = synth.disjoint_streams(P, N, int(0.6 * N) // P, seed=5)
    streams = [(i, np.random.default_rng(r).standard_normal(len(i))) for r, (i, _) in enumerate(streams)]
    outs = check(orc, P, N, streams, S.SSAR_SPLIT_ALLGATHER)
    assert not S.read_result(outs[0]).dense
    # past 2N/3: dense
    streams = synth.disjoint_streams(P, N, int(0.7 * N) // P, seed=6)
    streams = [(i, np.random.default_rng(r).standard_normal(len(i))) for r, (i, _) in enumerate(streams)]
    outs = check(orc, P, N, streams, S.SSAR_SPLIT_ALLGATHER)
    assert S.read_result(outs[0]).dense


def test_f64_empty_and_single(orc):
    N = 5000
    streams = [(np.zeros(0, np.uint32), np.zeros(0)), (np.array([4999], np.uint32), np.array([1.0 + 2.0 ** -40]))]
    for algo in ALGOS.values():
        check(orc, 2, N, streams, algo)


def test_f64_repeated_calls_one_world(orc):
    P, N = 4, 50_000
    w = S.LocalWorld(P, N, 20_000)
    for it, algo in enumerate(["ssar", "rd", "dsar", "auto", "ssar", "dsar"]):
        streams = synth.uniform_streams(P, N, 1000 + 3000 * it, seed=100 + it, kind="normal64")
        check(orc, P, N, streams, ALGOS[algo], world=w)


def test_f64_in_place(orc):
    P, N, k = 4, 80_000, 2000
    streams = synth.uniform_streams(P, N, k, seed=9, kind="normal64")
    w = S.LocalWorld(P, N, k)
    outs = [S.new_out(N, "cuda", torch.float64) for _ in range(P)]
    ins = []
    for o, (i, v) in zip(outs, streams):
        iv, vv = S.payload_views(o, N, len(i), torch.float64)
        iv.copy_(torch.from_numpy(i.view(np.int32)))
        vv.copy_(torch.from_numpy(v))
        ins.append((iv, vv))
    w.allreduce(ins, N, outs=outs, opts=S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER))
    torch.cuda.synchronize()
    res, _, _ = orc.split_allgather(N, streams, algo=orc.ALGO_SSAR_SPLIT, dtype=F64)
    for r in range(P):
        g = S.read_result(outs[r])
        np.testing.assert_array_equal(g.idx.cpu().numpy().view(np.uint32), res[r][1])
        np.testing.assert_array_equal(g.val.cpu().numpy(), res[r][2])


def test_f64_rejects_qsgd_and_small_out():
    w = S.LocalWorld(2, 1000, 100)
    s = [(torch.tensor([1], dtype=torch.int32, device="cuda"), torch.ones(1, dtype=torch.float64, device="cuda"))] * 2
    with pytest.raises(S.SparcmlError):
        w.allreduce(s, 1000, opts=S.make_opts(algo=S.DSAR_SPLIT_ALLGATHER, quant_bits=4))
    small = [S.new_out(1000, "cuda", torch.float32) for _ in range(2)]   # sized for fp32 values
    with pytest.raises(S.SparcmlError):
        w.allreduce(s, 1000, outs=small)


def test_apply_update_ignores_f64_results():
    w = S.LocalWorld(2, 1000, 10)
    s = [(torch.tensor([3], dtype=torch.int32, device="cuda"), torch.ones(1, dtype=torch.float64, device="cuda"))] * 2
    outs = w.allreduce(s, 1000)
    v = torch.ones(1000, device="cuda")
    S.apply_update(v, outs[0])
    torch.cuda.synchronize()
    assert torch.all(v == 1.0)


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("frac", [0.01, 0.3, 0.8])
def test_f64_sparse_allgather(orc, P, frac):
    # disjoint slices (SCD, R-27) with double values; dense past floor(N*8/12)
    N = 30_011
    bounds = np.linspace(0, N, P + 1).astype(np.int64)
    g = np.random.default_rng(P)
    streams = []
    for r in range(P):
        lo, hi = bounds[P - 1 - r], bounds[P - r]   # ranks in reverse range order
        n = int(frac * (hi - lo))
        streams.append((np.sort(g.choice(np.arange(lo, hi), n, replace=False)).astype(np.uint32),
                        g.standard_normal(n)))
    w = S.LocalWorld(P, N, max(1, max(len(s[0]) for s in streams)))
    outs = w.allgather(to_cuda(streams), N)
    torch.cuda.synchronize()
    ref, st = orc.sparse_allgather(N, streams, dtype=F64)
    for r in range(P):
        gr = S.read_result(outs[r])
        d, ei, ev = ref[r]
        assert gr.header.magic == S.HEADER_MAGIC_F64 and gr.header.status == 0
        assert gr.dense == bool(d)
        if d:
            np.testing.assert_array_equal(gr.val.cpu().numpy(), ev)
        else:
            np.testing.assert_array_equal(gr.idx.cpu().numpy().view(np.uint32), ei)
            np.testing.assert_array_equal(gr.val.cpu().numpy(), ev)
        if P > 1:
            assert gr.header.bytes_sent == st[r]["bytes_sent"] and gr.header.bytes_recv == st[r]["bytes_recv"]


@pytest.mark.parametrize("k", [50, 4000])   # sparse and dense (K > floor(8N/12)) results
def test_apply_update_f64(orc, k):
    P, N = 2, 5000
    streams = synth.uniform_streams(P, N, k, seed=k, kind="normal64")
    w = S.LocalWorld(P, N, k)
    outs = w.allreduce(to_cuda(streams), N)
    v0 = np.random.default_rng(1).standard_normal(N)
    v = torch.from_numpy(v0.copy()).cuda()
    S.apply_update(v, outs[0])
    v32 = torch.ones(N, device="cuda")
    S.apply_update(v32, outs[0])   # an fp64 result leaves an fp32 vector unchanged
    torch.cuda.synchronize()
    ref, _, _ = orc.split_allgather(N, streams, dtype=F64)
    np.testing.assert_array_equal(v.cpu().numpy(), orc.apply_update(v0, ref[0], N, dtype=F64))
    assert torch.all(v32 == 1.0)
