"""GPU parity of the stream kernels against the oracle, element by element,
through the C ABI: union-merge-with-sum, top-k (+EF) and the QSGD codec.
Sizes span several tiles plus ragged tails; integer/index outputs must be
bit-exact, and so must float values here (same operations, same order)."""
import numpy as np
import pytest

from paper_1802_08021_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1802_08021_b200 import sparcml as S  # noqa: E402


def cu(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dtype=dtype, device="cuda")


def cu_idx(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def host_idx(t):
    return t.cpu().numpy().view(np.uint32)


MERGE_CASES = [
    (0, 0, 100), (0, 5, 100), (7, 0, 100), (1, 1, 2), (2047, 1, 5000), (2048, 2048, 10_000),
    (3000, 5000, 9000), (10_000, 10_000, 10_000), (100_000, 30_000, 1 << 20), (70_001, 70_003, 1 << 18),
    (4095, 1, 9000), (4096, 4096, 20_000), (12_289, 4099, 30_000), (1_677_721, 1_677_721, 1 << 24),
]


@pytest.mark.parametrize("na,nb,N", MERGE_CASES)
def test_merge_sum_parity(orc, na, nb, N):
    (ia, va), (ib, vb) = synth.uniform_streams(2, N, [na, nb], seed=na + nb, kind="normal")
    io, vo = S.merge_sum(cu_idx(ia), cu(va, torch.float32), cu_idx(ib), cu(vb, torch.float32))
    eo, ev = orc.merge_sum(ia, va, ib, vb)
    np.testing.assert_array_equal(host_idx(io), eo)
    np.testing.assert_array_equal(vo.cpu().numpy().view(np.uint32), ev.view(np.uint32))


@pytest.mark.parametrize("off_a,off_b", [(1, 0), (0, 3), (2, 1), (4, 4)])
def test_merge_sum_unaligned_inputs(orc, off_a, off_b):
    """Streams starting at any 4-byte offset: the 16-byte staging loads apply only to aligned quads."""
    N = 1 << 17
    (ia, va), (ib, vb) = synth.uniform_streams(2, N, [9001 + off_a, 7003 + off_b], seed=5, kind="normal")
    ta, tva = cu_idx(ia), cu(va, torch.float32)
    tb, tvb = cu_idx(ib), cu(vb, torch.float32)
    io, vo = S.merge_sum(ta[off_a:], tva[off_a:], tb[off_b:], tvb[off_b:])
    eo, ev = orc.merge_sum(ia[off_a:], va[off_a:], ib[off_b:], vb[off_b:])
    np.testing.assert_array_equal(host_idx(io), eo)
    np.testing.assert_array_equal(vo.cpu().numpy().view(np.uint32), ev.view(np.uint32))


def test_merge_identical_and_disjoint(orc):
    N = 1 << 16
    for streams in (synth.identical_streams(2, N, 20_000, seed=1), synth.disjoint_streams(2, N, 20_000, seed=1)):
        (ia, va), (ib, vb) = streams
        io, vo = S.merge_sum(cu_idx(ia), cu(va, torch.float32), cu_idx(ib), cu(vb, torch.float32))
        eo, ev = orc.merge_sum(ia, va, ib, vb)
        np.testing.assert_array_equal(host_idx(io), eo)
        np.testing.assert_array_equal(vo.cpu().numpy(), ev)


TOPK_CASES = [
    (1, 1), (10, 3), (1000, 1), (4095, 17), (4097, 4096), (65_535, 100), (65_536, 655),
    (1 << 20, 1), (1 << 20, 1048), (1 << 20, 10_485), (3_000_001, 3000), (1 << 22, 41_943),
]


@pytest.mark.parametrize("N,k", TOPK_CASES)
def test_topk_parity(orc, N, k):
    x = synth.gaussian_vector(N, seed=N % 97 + k)
    xt = cu(x, torch.float32)
    res = torch.empty_like(xt)
    ws = S.TopkWorkspace(N, k)
    io, vo = S.topk_sparsify(xt, k, residual=res, ws=ws)
    ei, ev, er = orc.topk(x, k, residual=True)
    np.testing.assert_array_equal(host_idx(io), ei)
    np.testing.assert_array_equal(vo.cpu().numpy(), ev)
    np.testing.assert_array_equal(res.cpu().numpy(), er)
    st, passes = ws.status()
    assert st == 0 and passes in ((0, 1, 2) if k >= N else (1, 2))


def test_topk_ties_lower_index_wins(orc):
    rng = np.random.default_rng(3)
    for N, k in [(5000, 123), (300_000, 4_000), (1 << 20, 77_777)]:
        x = (rng.integers(-8, 9, size=N) * 0.5).astype(np.float32)   # massive ties
        io, vo = S.topk_sparsify(cu(x, torch.float32), k)
        ei, ev = orc.topk(x, k)
        np.testing.assert_array_equal(host_idx(io), ei)
        np.testing.assert_array_equal(vo.cpu().numpy(), ev)


def test_topk_sparse_input_and_in_place_residual(orc):
    N, k = 1 << 20, 5000
    x = np.zeros(N, np.float32)
    sel = np.random.default_rng(1).choice(N, 3000, replace=False)
    x[sel] = 1.0 + np.arange(3000, dtype=np.float32)   # fewer non-zeros than k: zeros fill in index order
    xt = cu(x, torch.float32)
    io, vo = S.topk_sparsify(xt, k, residual=xt)        # residual aliases x
    ei, ev, er = orc.topk(x, k, residual=True)
    np.testing.assert_array_equal(host_idx(io), ei)
    np.testing.assert_array_equal(vo.cpu().numpy(), ev)
    np.testing.assert_array_equal(xt.cpu().numpy(), er)


def _defeat_sample(N, rng, small, large):
    """Large values at exactly the granules the kernel samples, small ones elsewhere."""
    x = small(N)
    pos = S.topk_sample_positions(N).astype(np.int64)
    assert len(pos) > 1000
    for q in range(4):
        x[pos + q] = large(len(pos))
    return x, 4 * len(pos)


def test_topk_fallback_when_sample_underestimates(orc):
    """Adversarial input: every sampled granule holds large values, the rest are
    small, and k exceeds the number of large values.  The sampled threshold then
    admits fewer than k candidates and the kernel must take its exact re-filter
    path (passes == 2) and still be exact."""
    N, k = 1 << 20, 1 << 18
    rng = np.random.default_rng(5)
    x, nl = _defeat_sample(N, rng, lambda n: rng.random(n, dtype=np.float32),
                           lambda n: 100.0 + rng.random(n, dtype=np.float32) * 100.0)
    assert nl < k
    ws = S.TopkWorkspace(N, k)
    res = torch.empty(N, device="cuda")
    io, vo = S.topk_sparsify(cu(x, torch.float32), k, residual=res, ws=ws)
    ei, ev, er = orc.topk(x, k, residual=True)
    np.testing.assert_array_equal(host_idx(io), ei)
    np.testing.assert_array_equal(vo.cpu().numpy(), ev)
    np.testing.assert_array_equal(res.cpu().numpy(), er)
    assert ws.status() == (0, 2)


def test_ef_topk_fallback_when_sample_underestimates(orc):
    """The same with error feedback: the re-filter reads acc back from eps (which
    the kernel has already overwritten) and must still be exact."""
    N, k = 1 << 20, 1 << 17
    rng = np.random.default_rng(6)
    eps = (rng.random(N, dtype=np.float32) * np.float32(0.01)).astype(np.float32)
    g, nl = _defeat_sample(N, rng, lambda n: rng.standard_normal(n).astype(np.float32) * np.float32(0.1),
                           lambda n: np.float32(1000.0) + rng.random(n, dtype=np.float32))
    assert nl < k
    ws = S.TopkWorkspace(N, k)
    et = cu(eps, torch.float32)
    io, vo = S.ef_topk(et, cu(g, torch.float32), 0.5, k, ws=ws)
    ei, ev, ee = orc.ef_topk(eps, g, 0.5, k)
    np.testing.assert_array_equal(host_idx(io), ei)
    np.testing.assert_array_equal(vo.cpu().numpy(), ev)
    np.testing.assert_array_equal(et.cpu().numpy(), ee)
    assert ws.status() == (0, 2)


@pytest.mark.parametrize("ef,k", [(False, 1048), (True, 1048), (False, 100_000), (True, 300_000)])
def test_topk_sample_far_below_the_data(orc, ef, k):
    """Adversarial the other way: the sampled granules hold tiny values, every
    other value is normal, so the sampled threshold and histogram range sit far
    below the data -- every value is a candidate (spilled past the shared
    lists), all land in the overflow bin, and the refine levels of the slow path
    must still find the exact selection."""
    N = 1 << 20
    rng = np.random.default_rng(12)
    x, _ = _defeat_sample(N, rng, lambda n: rng.standard_normal(n).astype(np.float32),
                          lambda n: (rng.random(n, dtype=np.float32) * np.float32(1e-30)).astype(np.float32))
    ws = S.TopkWorkspace(N, k)
    if ef:
        g, _ = _defeat_sample(N, rng, lambda n: rng.standard_normal(n).astype(np.float32),
                              lambda n: (rng.random(n, dtype=np.float32) * np.float32(1e-30)).astype(np.float32))
        et = cu(x, torch.float32)
        io, vo = S.ef_topk(et, cu(g, torch.float32), 0.5, k, ws=ws)
        ei, ev, ee = orc.ef_topk(x, g, 0.5, k)
        np.testing.assert_array_equal(et.cpu().numpy(), ee)
    else:
        res = torch.empty(N, device="cuda")
        io, vo = S.topk_sparsify(cu(x, torch.float32), k, residual=res, ws=ws)
        ei, ev, er = orc.topk(x, k, residual=True)
        np.testing.assert_array_equal(res.cpu().numpy(), er)
    np.testing.assert_array_equal(host_idx(io), ei)
    np.testing.assert_array_equal(vo.cpu().numpy(), ev)
    assert ws.status()[0] == 0


def test_topk_workspace_reused_across_sizes(orc):
    """One workspace, zeroed once, serves calls at any N up to its size, in any
    order (every histogram slot is cleared by the call that used it)."""
    ws = S.TopkWorkspace(300_000, 3000)
    rng = np.random.default_rng(8)
    for it, (N, k, ef) in enumerate([(1000, 10, False), (10_000, 100, True), (300_000, 3000, False),
                                     (1000, 999, True), (70_000, 700, True), (10_000, 1, False),
                                     (1000, 10, False), (300_000, 2999, True), (4096, 4095, False)]):
        x = rng.standard_normal(N).astype(np.float32)
        if ef:
            g = rng.standard_normal(N).astype(np.float32)
            et = cu(x, torch.float32)
            io, vo = S.ef_topk(et, cu(g, torch.float32), 0.25, k, ws=ws)
            ei, ev, ee = orc.ef_topk(x, g, 0.25, k)
            np.testing.assert_array_equal(et.cpu().numpy(), ee)
        else:
            io, vo = S.topk_sparsify(cu(x, torch.float32), k, ws=ws)
            ei, ev = orc.topk(x, k)
        np.testing.assert_array_equal(host_idx(io), ei, err_msg=f"call {it}")
        np.testing.assert_array_equal(vo.cpu().numpy(), ev, err_msg=f"call {it}")
        assert ws.status() == (0, 1)


@pytest.mark.parametrize("ef", [False, True])
def test_topk_warm_start_hits_and_misses_are_exact(orc, ef):
    """A call on a workspace whose previous call had the same (N, k) takes tau
    and the histogram range from that call's k-th magnitude instead of sampling.
    Same distribution: a hit (one pass).  Data scaled by 1e-3: every value is
    below the warm tau, so the exact re-filter runs (passes == 2, which a
    sampled tau would not need -- the warm start was taken).  The next call
    samples again.  Data scaled by 1e3: the k-th magnitude lies above the
    histogram range (the overflow bin's refinement).  All bit-exact."""
    N, k = 1 << 20, 10_000
    ws = S.TopkWorkspace(N, k)
    rng = np.random.default_rng(21)
    expect_passes = [1, 1, 2, 1, 1, 1, 1]
    for it, (scale, want) in enumerate(zip([1.0, 1.0, 1e-3, 1.0, 1.0, 1e3, 1.0], expect_passes)):
        x = (rng.standard_normal(N) * scale).astype(np.float32)
        if ef:
            g = (rng.standard_normal(N) * scale).astype(np.float32)
            et = cu(x, torch.float32)
            io, vo = S.ef_topk(et, cu(g, torch.float32), 0.5, k, ws=ws)
            ei, ev, ee = orc.ef_topk(x, g, 0.5, k)
            np.testing.assert_array_equal(et.cpu().numpy(), ee, err_msg=f"call {it}")
        else:
            res = torch.empty(N, device="cuda")
            io, vo = S.topk_sparsify(cu(x, torch.float32), k, residual=res, ws=ws)
            ei, ev, er = orc.topk(x, k, residual=True)
            np.testing.assert_array_equal(res.cpu().numpy(), er, err_msg=f"call {it}")
        np.testing.assert_array_equal(host_idx(io), ei, err_msg=f"call {it}")
        np.testing.assert_array_equal(vo.cpu().numpy(), ev, err_msg=f"call {it}")
        assert ws.status() == (0, want), f"call {it}"


def test_ef_topk_warm_start_over_many_steps(orc):
    """Algorithm 1's loop for 12 steps on one workspace: from the
    second step on tau comes from the previous step's k-th magnitude, which
    drifts upward while the accumulator fills (the early steps can land in the
    overflow bin).  Every step bit-exact, eps included."""
    N, k = 1 << 19, 5243
    eps = np.zeros(N, np.float32)
    grads = [synth.gaussian_vector(N, seed=40 + s) for s in range(3)]
    et = torch.zeros(N, device="cuda")
    gts = [cu(g, torch.float32) for g in grads]
    ws = S.TopkWorkspace(N, k)
    for step in range(12):
        io, vo = S.ef_topk(et, gts[step % 3], 0.01, k, ws=ws)
        ei, ev, eps = orc.ef_topk(eps, grads[step % 3], 0.01, k)
        np.testing.assert_array_equal(host_idx(io), ei, err_msg=f"step {step}")
        np.testing.assert_array_equal(vo.cpu().numpy(), ev, err_msg=f"step {step}")
        np.testing.assert_array_equal(et.cpu().numpy(), eps, err_msg=f"step {step}")
        assert ws.status()[0] == 0


def test_topk_heavy_ties_refine_levels(orc):
    """Half-integer values (config 5's gradients) give crossing bins of one
    magnitude with far more than the list capacity: exact-bin and refine paths."""
    rng = np.random.default_rng(11)
    for N, k in [(1 << 20, 100_000), (3_231_961, 32_319), (1 << 22, 1_000_000)]:
        x = (rng.integers(-40, 41, size=N) * 0.5).astype(np.float32)
        io, vo = S.topk_sparsify(cu(x, torch.float32), k)
        ei, ev = orc.topk(x, k)
        np.testing.assert_array_equal(host_idx(io), ei)
        np.testing.assert_array_equal(vo.cpu().numpy(), ev)


def test_topk_nonfinite_reported():
    x = synth.gaussian_vector(1 << 17, seed=9)
    x[777] = np.inf
    ws = S.TopkWorkspace(len(x), 100)
    S.topk_sparsify(cu(x, torch.float32), 100, ws=ws)
    assert ws.status()[0] == S.ERR_NONFINITE
    x[777] = 1.0
    S.topk_sparsify(cu(x, torch.float32), 100, ws=ws)
    assert ws.status()[0] == 0


def test_topk_k_ge_n(orc):
    x = synth.gaussian_vector(1000, seed=2)
    io, vo = S.topk_sparsify(cu(x, torch.float32), 5000)
    np.testing.assert_array_equal(host_idx(io), np.arange(1000))
    np.testing.assert_array_equal(vo.cpu().numpy(), x)


@pytest.mark.parametrize("N,k", [(100_000, 100), (1 << 21, 2097), (25_557_032 // 8, 3194)])
def test_ef_topk_parity(orc, N, k):
    eps = synth.gaussian_vector(N, seed=5) * np.float32(0.1)
    g = synth.gaussian_vector(N, seed=6)
    et = cu(eps, torch.float32)
    gt = cu(g, torch.float32)
    ws = S.TopkWorkspace(N, k)
    for step in range(3):   # error feedback carries over steps
        io, vo = S.ef_topk(et, gt, 0.05, k, ws=ws)
        ei, ev, eps = orc.ef_topk(eps, g, 0.05, k)
        np.testing.assert_array_equal(host_idx(io), ei)
        np.testing.assert_array_equal(vo.cpu().numpy(), ev)
        np.testing.assert_array_equal(et.cpu().numpy(), eps)


@pytest.mark.parametrize("n", [1, 7, 8, 1000, 1024, 4099, 1 << 20, 1_000_003])
@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("B", [8, 256, 1024])
def test_qsgd_parity(orc, n, bits, B):
    x = synth.gaussian_vector(n, seed=n + bits)
    seed, base = 1234 + bits, 3 * n + 5
    c, s = S.quantize(cu(x, torch.float32), bits, bucket=B, seed=seed, ctr_base=base)
    ec, es = orc.qsgd_quantize(x, bits, bucket=B, seed=seed, ctr_base=base)
    np.testing.assert_array_equal(c.cpu().numpy(), ec)
    np.testing.assert_array_equal(s.cpu().numpy(), es)
    d = S.dequantize(c.clone(), s, n, bits, bucket=B)
    np.testing.assert_array_equal(d.cpu().numpy(), orc.qsgd_dequantize(ec, es, n, bits, B))


# ---- bucketed top-k (§7; reading R-26) -------------------
BUCKET_CASES = [
    (512, 4, 512), (513, 4, 512), (1 << 20, 4, 512), (1 << 20, 16, 512), (1_000_003, 8, 512),
    (100_000, 2, 128), (100_000, 50, 384), (300_001, 100, 1024), (70_000, 1024, 1024), (5000, 700, 512),
    (129, 1, 128), (1, 1, 128),
]


@pytest.mark.parametrize("N,k,B", BUCKET_CASES)
def test_topk_bucketed_parity(orc, N, k, B):
    x = synth.gaussian_vector(N, seed=N % 89 + k + B)
    xt = cu(x, torch.float32)
    res = torch.empty_like(xt)
    io, vo = S.topk_sparsify(xt, k, residual=res, bucket=B)
    ei, ev, er = orc.topk_bucketed(x, k, B, residual=True)
    np.testing.assert_array_equal(host_idx(io), ei)
    np.testing.assert_array_equal(vo.cpu().numpy(), ev)
    np.testing.assert_array_equal(res.cpu().numpy(), er)


def test_topk_bucketed_ties_and_in_place(orc):
    rng = np.random.default_rng(12)
    for N, k, B in [(4096, 5, 512), (200_003, 17, 256), (1 << 20, 8, 1024)]:
        x = (rng.integers(-4, 5, size=N) * 0.5).astype(np.float32)   # massive ties, zeros
        xt = cu(x, torch.float32)
        io, vo = S.topk_sparsify(xt, k, residual=xt, bucket=B)        # residual aliases x
        ei, ev, er = orc.topk_bucketed(x, k, B, residual=True)
        np.testing.assert_array_equal(host_idx(io), ei)
        np.testing.assert_array_equal(vo.cpu().numpy(), ev)
        np.testing.assert_array_equal(xt.cpu().numpy(), er)


@pytest.mark.parametrize("N,k,B", [(1 << 20, 4, 512), (25_557_032 // 16, 8, 512), (99_999, 3, 128)])
def test_ef_topk_bucketed_parity(orc, N, k, B):
    eps = synth.gaussian_vector(N, seed=15) * np.float32(0.1)
    g = synth.gaussian_vector(N, seed=16)
    et, gt = cu(eps, torch.float32), cu(g, torch.float32)
    ws = S.TopkWorkspace(N, k)
    for step in range(3):
        io, vo = S.ef_topk(et, gt, 0.05, k, bucket=B, ws=ws)
        ei, ev, eps = orc.ef_topk_bucketed(eps, g, 0.05, k, B)
        np.testing.assert_array_equal(host_idx(io), ei)
        np.testing.assert_array_equal(vo.cpu().numpy(), ev)
        np.testing.assert_array_equal(et.cpu().numpy(), eps)
        assert ws.status() == (0, 1)


def test_topk_bucketed_nonfinite_reported():
    x = synth.gaussian_vector(1 << 16, seed=19)
    x[4321] = np.nan
    ws = S.TopkWorkspace(len(x), 4)
    S.topk_sparsify(cu(x, torch.float32), 4, ws=ws, bucket=512)
    assert ws.status()[0] == S.ERR_NONFINITE
    x[4321] = 0.5
    S.topk_sparsify(cu(x, torch.float32), 4, ws=ws, bucket=512)
    assert ws.status()[0] == 0


@pytest.mark.parametrize("n", [7, 1000, 4099, 1 << 20])
@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("B", [8, 128, 256, 1024])
def test_qsgd_l2_parity(orc, n, bits, B):
    """l2-norm scale (reading R-31): the fixed balanced tree makes codes and
    scales bit-exact against the oracle."""
    x = synth.gaussian_vector(n, seed=3 * n + bits + B)
    c, s = S.quantize(cu(x, torch.float32), bits, bucket=B, seed=77, ctr_base=5, norm=1)
    with orc.qsgd_norm_scope(1):
        ec, es = orc.qsgd_quantize(x, bits, bucket=B, seed=77, ctr_base=5)
    np.testing.assert_array_equal(s.cpu().numpy(), es)
    np.testing.assert_array_equal(c.cpu().numpy(), ec)


@pytest.mark.parametrize("N,k,bucket", [(1 << 24, 167_772, 0), (25_557_032, 25_557, 0), (25_557_032, 4, 512),
                                         (1 << 24, 1_677_721, 0)])
def test_topk_bench_sizes(orc, N, k, bucket):
    """The bench's top-k launches at full size (cfg2, cfg3, bucket512, cfg4's 10 %): EF over
    two steps, bit-exact indices, values and residual against the oracle."""
    g = synth.gaussian_vector(N, seed=0)
    eps = np.zeros(N, np.float32)
    et, gt = cu(eps, torch.float32), cu(g, torch.float32)
    ws = S.TopkWorkspace(N, k if bucket == 0 else 1)
    for step in range(2):
        io, vo = S.ef_topk(et, gt, 0.01, k, ws=ws, bucket=bucket)
        if bucket:
            ei, ev, eps = orc.ef_topk_bucketed(eps, g, 0.01, k, bucket)
        else:
            ei, ev, eps = orc.ef_topk(eps, g, 0.01, k)
        np.testing.assert_array_equal(host_idx(io), ei)
        np.testing.assert_array_equal(vo.cpu().numpy(), ev)
        np.testing.assert_array_equal(et.cpu().numpy(), eps)
