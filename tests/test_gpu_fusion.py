"""NEXT row 1: layer-wise tensor fusion on a loopback world.
L layers laid end to end are fused into one stream (index offsets), reduced
by ONE allreduce and split back by index range; every layer must equal the
oracle's per-layer allreduce (the summation tree is over ranks, reading R-8,
so fusion cannot change a value), and the fused result must equal the
oracle's allreduce of the fused streams."""
import numpy as np
import pytest

from paper_1802_08021_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1802_08021_b200 import sparcml as S  # noqa: E402


def _dense(res, N, off=0, idx=None, val=None):
    got = np.zeros(N, np.float32)
    mask = np.ones(N, np.uint8)
    if idx is None:
        got[:] = val
    else:
        ii = idx.astype(np.int64) - off
        got[ii] = val
        mask[:] = 0
        mask[ii] = 1
    return mask, got


@pytest.mark.parametrize("P,algo", [(4, S.SSAR_SPLIT_ALLGATHER), (3, S.SSAR_SPLIT_ALLGATHER),
                                    (4, S.SSAR_RECURSIVE_DOUBLE), (2, S.DSAR_SPLIT_ALLGATHER)])
def test_fused_layers_match_per_layer_oracle(orc, P, algo):
    dims = [100_003, 1_000_000, 777, 16, 250_000]
    ks = [1000, 9000, 50, 1, 2500]
    off = S.layer_offsets(dims)
    layers = [synth.uniform_streams(P, dims[l], ks[l], seed=70 + l, kind="normal") for l in range(len(dims))]
    w = S.LocalWorld(P, off[-1], sum(ks))
    fused = []
    for r in range(P):
        mine = [(torch.from_numpy(layers[l][r][0].view(np.int32)).cuda(), torch.from_numpy(layers[l][r][1]).cuda())
                for l in range(len(dims))]
        fused.append(S.fuse_streams(mine, off))
    outs = w.allreduce(fused, off[-1], opts=S.make_opts(algo=algo))
    # the fused streams are exactly the concatenation with offsets
    for r in range(P):
        want_i = np.concatenate([layers[l][r][0].astype(np.int64) + off[l] for l in range(len(dims))])
        np.testing.assert_array_equal(fused[r][0].cpu().numpy().view(np.uint32), want_i)
    oa = orc.ALGO_SSAR_SPLIT if algo != S.DSAR_SPLIT_ALLGATHER else orc.ALGO_DSAR_SPLIT
    fused_host = [(fused[r][0].cpu().numpy().view(np.uint32), fused[r][1].cpu().numpy()) for r in range(P)]
    if algo == S.SSAR_RECURSIVE_DOUBLE:
        ref_f, _ = orc.ssar_recursive_double(off[-1], fused_host)
    else:
        ref_f, _, _ = orc.split_allgather(off[-1], fused_host, algo=oa)
    for r in range(P):
        res = S.read_result(outs[r])
        mf, vf = orc.result_to_dense(ref_f[r], off[-1])
        mg, vg = _dense(res, off[-1], idx=None if res.dense else res.idx.cpu().numpy().view(np.uint32),
                        val=res.val.cpu().numpy())
        np.testing.assert_array_equal(vg, vf)
        np.testing.assert_array_equal(mg, mf)
        parts = S.split_result(outs[r], off)
        for l in range(len(dims)):
            ref, _, _ = orc.split_allgather(dims[l], layers[l], algo=orc.ALGO_SSAR_SPLIT)
            wm, wv = orc.result_to_dense(ref[r], dims[l])
            pi, pv = parts[l]
            gm, gv = _dense(None, dims[l], off[l], None if pi is None else pi.cpu().numpy().view(np.uint32),
                            pv.cpu().numpy())
            np.testing.assert_array_equal(gv, wv)
            if pi is not None:
                np.testing.assert_array_equal(gm, wm)


def test_layer_ranges_sparse_and_dense():
    N = 1000
    off = [0, 100, 100, 640, N]
    idx = torch.tensor([3, 99, 100, 101, 639, 640, 999], dtype=torch.int32, device="cuda")
    val = torch.arange(7, dtype=torch.float32, device="cuda") + 1
    w = S.LocalWorld(1, N, 16)
    out = w.allreduce([(idx, val)], N, opts=S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER))[0]
    r = S.layer_ranges(out, off).cpu().tolist()
    assert r == [0, 2, 2, 5, 7]
    out2 = w.allreduce([(idx, val)], N, opts=S.make_opts(algo=S.DSAR_SPLIT_ALLGATHER))[0]
    assert S.layer_ranges(out2, off).cpu().tolist() == [0, 100, 100, 640, N]
