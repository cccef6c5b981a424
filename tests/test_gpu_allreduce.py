"""GPU parity of the sparse allreduce against the oracle's simulators.

A loopback world runs all P ranks' kernels and exchanges on one GPU through
the same code path the multi-process (CUDA IPC) world uses, except that the
peer pointers are local and the flag barrier does not wait.  For every rank:
representation flag, nnz and indices bit-exact; values bit-exact (the GPU
follows the same summation tree, R-8), which implies north_star's
1e-5 relative bar; header accounting equal to the oracle's trace."""
import numpy as np
import pytest

from paper_1802_08021_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1802_08021_b200 import sparcml as S  # noqa: E402

ALGOS = {"rd": S.SSAR_RECURSIVE_DOUBLE, "ssar": S.SSAR_SPLIT_ALLGATHER, "dsar": S.DSAR_SPLIT_ALLGATHER,
         "auto": S.ALGO_AUTO}


def to_cuda(streams):
    out = []
    for i, v in streams:
        out.append((torch.from_numpy(np.ascontiguousarray(i, np.uint32).view(np.int32)).cuda(),
                    torch.from_numpy(np.ascontiguousarray(v, np.float32)).cuda()))
    return out


def oracle_run(orc, N, streams, algo, bits=0, bucket=1024, seed=0):
    if algo == S.SSAR_RECURSIVE_DOUBLE:
        res, st = orc.ssar_recursive_double(N, streams)
        return res, st, False
    oalgo = {S.SSAR_SPLIT_ALLGATHER: orc.ALGO_SSAR_SPLIT, S.DSAR_SPLIT_ALLGATHER: orc.ALGO_DSAR_SPLIT,
             S.ALGO_AUTO: orc.ALGO_AUTO}[algo]
    return orc.split_allgather(N, streams, algo=oalgo, quant_bits=bits, bucket=bucket, seed=seed)


def check_world(orc, P, N, streams, algo, bits=0, bucket=1024, seed=0, world=None, expect_algo=None):
    w = world or S.LocalWorld(P, N, max(1, max(len(s[0]) for s in streams)))
    opts = S.make_opts(algo=algo, quant_bits=bits, quant_bucket=bucket, seed=seed)
    outs = w.allreduce(to_cuda(streams), N, opts=opts)
    torch.cuda.synchronize()
    oalgo = algo   # AUTO: split-allgather at every size (the measured crossover, csrc/api.cu kRdMaxBytes)
    res, st, _ = oracle_run(orc, N, streams, oalgo if P > 1 else (S.ALGO_AUTO if algo == S.SSAR_RECURSIVE_DOUBLE else algo),
                            bits, bucket, seed)
    for r in range(P):
        g = S.read_result(outs[r])
        d, ei, ev = res[r]
        assert g.header.magic == S.HEADER_MAGIC
        assert g.header.status == 0
        assert g.header.N == N
        assert g.header.k_sum == sum(len(s[0]) for s in streams)
        assert g.dense == bool(d), f"rank {r}: representation differs"
        if d:
            np.testing.assert_array_equal(g.val.cpu().numpy(), ev)
        else:
            assert g.header.nnz == len(ei)
            np.testing.assert_array_equal(g.idx.cpu().numpy().view(np.uint32), ei)
            np.testing.assert_array_equal(g.val.cpu().numpy(), ev)
        if P > 1:
            assert g.header.bytes_recv == st[r]["bytes_recv"], f"rank {r} bytes_recv"
            assert g.header.bytes_sent == st[r]["bytes_sent"], f"rank {r} bytes_sent"
    return outs


@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7, 8, 12])
@pytest.mark.parametrize("d", [0.001, 0.01, 0.1, 0.3])
def test_rd(orc, P, d):
    N = 100_003
    k = max(1, int(d * N))
    streams = synth.uniform_streams(P, N, k, seed=int(d * 1000) + P, kind="normal")
    check_world(orc, P, N, streams, S.SSAR_RECURSIVE_DOUBLE)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 6, 8, 16])
@pytest.mark.parametrize("algo", ["ssar", "dsar", "auto"])
def test_split(orc, P, algo):
    N = 65_536 + 17 * P
    k = 4000
    streams = synth.uniform_streams(P, N, k, seed=P * 7, kind="normal")
    check_world(orc, P, N, streams, ALGOS[algo])


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("bits", [2, 4, 8])
def test_dsar_qsgd(orc, P, bits):
    """Codes depend on the pre-quantization sums: bit-exact sums (same tree)
    make the decoded result bit-exact too (reading R-16)."""
    N = 1 << 18
    streams = synth.uniform_streams(P, N, N // 5, seed=P + bits, kind="normal")
    check_world(orc, P, N, streams, S.DSAR_SPLIT_ALLGATHER, bits=bits, bucket=1024, seed=99)
    check_world(orc, P, N, streams, S.DSAR_SPLIT_ALLGATHER, bits=bits, bucket=64, seed=7)


def test_edge_cases(orc):
    # empty inputs on some ranks, all empty, a single shared index, dense from the start
    N = 5000
    e = (np.zeros(0, np.uint32), np.zeros(0, np.float32))
    one = (np.array([4999], np.uint32), np.array([2.5], np.float32))
    for P in [2, 3, 4, 5]:
        for algo in ["rd", "ssar", "dsar"]:
            check_world(orc, P, N, [e] * P, ALGOS[algo])
            check_world(orc, P, N, [one] + [e] * (P - 1), ALGOS[algo])
            check_world(orc, P, N, [one] * P, ALGOS[algo])
            full = (np.arange(N, dtype=np.uint32), np.ones(N, np.float32))
            check_world(orc, P, N, [full] * P, ALGOS[algo])


@pytest.mark.parametrize("P,frac", [(2, 0.6), (4, 0.3), (3, 0.9)])
def test_ssar_dense_block_ranges(orc, P, frac):
    """Forced SSAR on dense inputs: an owner block's window range holds more
    elements than one shared-memory tile, so it is reduced in pieces through
    the spill area (and K > delta makes the concatenation densify)."""
    N = 1 << 20
    streams = synth.uniform_streams(P, N, int(frac * N), seed=P + 31, kind="normal")
    check_world(orc, P, N, streams, S.SSAR_SPLIT_ALLGATHER)


def test_integer_values_exact_vs_definition(orc):
    """Integer-valued inputs: any summation order is exact, so the result must
    equal the plain definition (brute-force dense sum) bit for bit."""
    P, N = 8, 200_000
    streams = synth.uniform_streams(P, N, 20_000, seed=11, kind="int")
    bf = orc.brute_force(N, streams)
    w = S.LocalWorld(P, N, 20_000)
    for algo in ["rd", "ssar", "auto"]:
        outs = w.allreduce(to_cuda(streams), N, opts=S.make_opts(algo=ALGOS[algo]))
        for r in range(P):
            g = S.read_result(outs[r])
            if g.dense:
                np.testing.assert_array_equal(g.val.cpu().numpy(), bf["f32"])
            else:
                np.testing.assert_array_equal(g.idx.cpu().numpy().view(np.uint32), bf["idx"])
                np.testing.assert_array_equal(g.val.cpu().numpy().astype(np.float64), bf["d64"][bf["idx"]])


def test_repeated_calls_reuse_buffers(orc):
    """Back-to-back collectives on one world (buffer reuse across calls)."""
    P, N = 4, 1 << 16
    w = S.LocalWorld(P, N, 5000)
    for it in range(6):
        algo = [S.SSAR_RECURSIVE_DOUBLE, S.SSAR_SPLIT_ALLGATHER, S.DSAR_SPLIT_ALLGATHER][it % 3]
        streams = synth.uniform_streams(P, N, 1000 + 500 * it, seed=it, kind="normal")
        check_world(orc, P, N, streams, algo, world=w)


def test_validate_flags_unsorted(orc):
    P, N = 2, 1000
    bad = (np.array([5, 3, 9], np.uint32), np.ones(3, np.float32))
    good = (np.array([1, 2], np.uint32), np.ones(2, np.float32))
    w = S.LocalWorld(P, N, 10)
    outs = w.allreduce(to_cuda([bad, good]), N, opts=S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER, validate=True))
    assert S.read_result(outs[0]).header.status == S.ERR_UNSORTED
    outs = w.allreduce(to_cuda([good, good]), N, opts=S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER, validate=True))
    assert S.read_result(outs[0]).header.status == 0


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_baseline_configs_full_size(orc, cfg):
    """BASELINE.json configs at full size on a loopback world of P ranks
    (P = 8 except config 1), checked against the oracle element by element."""
    if cfg == "cfg1":
        P, N = 4, 4096
        streams = synth.uniform_streams(P, N, 64, seed=1)
        algo = S.SSAR_RECURSIVE_DOUBLE
    elif cfg == "cfg2":
        P, N = 8, 1 << 24
        streams = synth.uniform_streams(P, N, synth.k_for_density(N, 0.01), seed=2)
        algo = S.SSAR_SPLIT_ALLGATHER
    elif cfg == "cfg3":
        P, N, k = 8, 25_557_032, 25_557
        streams = []
        for r in range(P):
            i, v = orc.topk(synth.gaussian_vector(N, seed=3, rank=r), k)
            streams.append((i, v))
        algo = S.SSAR_RECURSIVE_DOUBLE
    elif cfg == "cfg4":
        P, N = 8, 1 << 24
        streams = synth.uniform_streams(P, N, synth.k_for_density(N, 0.10), seed=4)
        check_world(orc, P, N, streams, S.ALGO_AUTO, bits=4, seed=5)   # AUTO -> DSAR at P=8
        return
    else:
        P, N = 8, 3_231_961
        streams = synth.lr_gradient_streams(P, N, seed=5)
        algo = S.ALGO_AUTO
    check_world(orc, P, N, streams, algo)


@pytest.mark.parametrize("op", [S.OP_MAX, S.OP_MIN])
@pytest.mark.parametrize("P,algo", [(1, "ssar"), (1, "dsar"), (2, "rd"), (3, "rd"), (4, "ssar"), (5, "ssar"),
                                    (4, "dsar"), (3, "dsar"), (8, "auto")])
def test_max_min_operators(orc, op, P, algo):
    """MAX / MIN (reading R-30) on every algorithm: bit-exact against the
    oracle's simulators run with the same operator (neutral -inf / +inf in
    dense results), sparse and densifying cases."""
    for N, k in [(50_000, 500), (20_000, 6_000)]:
        streams = synth.uniform_streams(P, N, k, seed=op * 100 + P, kind="normal")
        w = S.LocalWorld(P, N, k)
        outs = w.allreduce(to_cuda(streams), N, opts=S.make_opts(algo=ALGOS[algo]), op=op)
        with orc.op_scope(op):
            oalgo = ALGOS[algo]
            res, st, _ = oracle_run(orc, N, streams, oalgo if P > 1 else ALGOS[algo])
        for r in range(P):
            g = S.read_result(outs[r])
            d, ei, ev = res[r]
            assert g.header.status == 0 and g.dense == bool(d)
            if d:
                np.testing.assert_array_equal(g.val.cpu().numpy(), ev)
            else:
                np.testing.assert_array_equal(g.idx.cpu().numpy().view(np.uint32), ei)
                np.testing.assert_array_equal(g.val.cpu().numpy(), ev)


def test_max_rejects_quantization():
    w = S.LocalWorld(2, 1000, 10)
    i = torch.arange(10, dtype=torch.int32, device="cuda")
    v = torch.ones(10, device="cuda")
    with pytest.raises(S.SparcmlError):
        w.allreduce([(i, v), (i, v)], 1000, opts=S.make_opts(algo=S.DSAR_SPLIT_ALLGATHER, quant_bits=4), op=S.OP_MAX)


@pytest.mark.parametrize("P,bits,B", [(1, 4, 1024), (2, 4, 1024), (4, 8, 256), (3, 2, 64)])
def test_dsar_qsgd_l2(orc, P, bits, B):
    """DSAR with the l2-norm QSGD scale (R-31), bit-exact against the oracle."""
    N = 1 << 18
    streams = synth.uniform_streams(P, N, N // 5, seed=P + bits + 40, kind="normal")
    w = S.LocalWorld(P, N, N // 5)
    opts = S.make_opts(algo=S.DSAR_SPLIT_ALLGATHER, quant_bits=bits, quant_bucket=B, seed=9, quant_norm=1)
    outs = w.allreduce(to_cuda(streams), N, opts=opts)
    with orc.qsgd_norm_scope(1):
        res, _, _ = orc.split_allgather(N, streams, algo=orc.ALGO_DSAR_SPLIT, quant_bits=bits, bucket=B, seed=9)
    for r in range(P):
        g = S.read_result(outs[r])
        assert g.dense and g.header.status == 0
        np.testing.assert_array_equal(g.val.cpu().numpy(), res[r][2])


@pytest.mark.parametrize("P,algo", [(1, "ssar"), (1, "auto"), (1, "dsar"), (4, "ssar"), (3, "dsar"), (2, "auto")])
def test_in_place_inputs(orc, P, algo):
    """Inputs written into the result's own payload slots (include/sparcml.h,
    in place): identical results to separate buffers; P = 1 then only writes
    the header."""
    N = 200_003
    streams = synth.uniform_streams(P, N, 3000 if algo != "dsar" else 60_000, seed=P + 70, kind="normal")
    w = S.LocalWorld(P, N, max(len(s[0]) for s in streams))
    outs = [S.new_out(N) for _ in range(P)]
    ins = []
    for r, (i, v) in enumerate(streams):
        vi, vv = S.payload_views(outs[r], N, len(i))
        vi.copy_(torch.from_numpy(i.view(np.int32)))
        vv.copy_(torch.from_numpy(v))
        ins.append((vi, vv))
    opts = S.make_opts(algo=ALGOS[algo])
    if algo == "auto" and P == 2:
        opts = S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER)
    w.allreduce(ins, N, outs=outs, opts=opts)
    ref, _, _ = oracle_run(orc, N, streams, ALGOS[algo] if algo != "auto" else S.ALGO_AUTO)
    for r in range(P):
        g = S.read_result(outs[r])
        d, ei, ev = ref[r]
        assert g.header.status == 0 and g.dense == bool(d)
        if d:
            np.testing.assert_array_equal(g.val.cpu().numpy(), ev)
        else:
            np.testing.assert_array_equal(g.idx.cpu().numpy().view(np.uint32), ei)
            np.testing.assert_array_equal(g.val.cpu().numpy(), ev)


def test_in_place_rejected_where_unsafe():
    N = 10_000
    w = S.LocalWorld(2, N, 100)
    outs = [S.new_out(N) for _ in range(2)]
    ins = []
    for r in range(2):
        vi, vv = S.payload_views(outs[r], N, 100)
        vi.copy_(torch.arange(100, dtype=torch.int32) * 7 + r)
        vv.fill_(1.0)
        ins.append((vi, vv))
    with pytest.raises(S.SparcmlError):
        w.allreduce(ins, N, outs=outs, opts=S.make_opts(algo=S.SSAR_RECURSIVE_DOUBLE))
    w1 = S.LocalWorld(1, 100, 100)
    o = S.new_out(100)
    vi, vv = S.payload_views(o, 100, 60)
    vi.copy_(torch.arange(60, dtype=torch.int32))
    vv.fill_(2.0)
    with pytest.raises(S.SparcmlError):   # 60 > delta = 50 under forced SSAR
        w1.allreduce([(vi, vv)], 100, outs=[o], opts=S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER))


@pytest.mark.parametrize("P,N,k", [(2, 4096, 16), (4, 4096, 64), (4, 1 << 16, 4096), (8, 1 << 20, 1000)])
def test_auto_follows_measured_crossover(orc, P, N, k):
    """AUTO picks recursive doubling only under the crossover measured on the box
    (csrc/api.cu kRdMaxBytes, profiles/r02_auto_crossover_p*.log): on 2 and 4 B200
    split-allgather won at every size, so AUTO runs split-allgather even for the
    smallest data (the paper's small-data rule, measured, not assumed)."""
    streams = synth.uniform_streams(P, N, k, seed=N + P)
    w = S.LocalWorld(P, N, k)
    outs = w.allreduce(to_cuda(streams), N, opts=S.make_opts(algo=S.ALGO_AUTO))
    ref, _, _ = orc.split_allgather(N, streams, algo=orc.ALGO_AUTO)
    for r in range(P):
        g = S.read_result(outs[r])
        assert g.header.status == 0
        assert g.header.algo_used in (S.SSAR_SPLIT_ALLGATHER, S.DSAR_SPLIT_ALLGATHER)
        d, ei, ev = ref[r]
        assert g.dense == bool(d)
        if not d:
            np.testing.assert_array_equal(g.idx.cpu().numpy().view(np.uint32), ei)
            np.testing.assert_array_equal(g.val.cpu().numpy(), ev)
    w.close()


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("algo", ["ssar", "auto"])
def test_split_three_kernel_path(orc, P, algo, monkeypatch):
    """SSAR known on the host runs the fused split-allgather kernel; the
    three-kernel path (push, owner, concat: what runs when the device decides
    SSAR/DSAR) stays bit-exact too (SPARCML_FUSED=0 selects it)."""
    monkeypatch.setenv("SPARCML_FUSED", "0")
    N = 70_001
    streams = synth.uniform_streams(P, N, 3000, seed=P + 50, kind="normal")
    check_world(orc, P, N, streams, ALGOS[algo])
    streams = synth.uniform_streams(P, N, 20_000, seed=P + 51, kind="normal")   # dense block ranges
    check_world(orc, P, N, streams, S.SSAR_SPLIT_ALLGATHER)


@pytest.mark.parametrize("P", [2, 3, 4, 8, 16])
def test_fused_split_back_to_back(orc, P):
    """Many fused calls on one world with changing sizes and densities: the
    arrival counters carry over between calls without a reset."""
    N = 90_000
    w = S.LocalWorld(P, N, 30_000)
    for it, k in enumerate([10, 3000, 30_000, 0, 1, 12_000, 500]):
        streams = synth.uniform_streams(P, N, k, seed=100 * P + it, kind="normal")
        check_world(orc, P, N, streams, S.SSAR_SPLIT_ALLGATHER, world=w)
    w.close()
