"""CPU oracle for the SparCML hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1802_08021_b200``) never imports it; the two share no code.

This module is argument marshalling (numpy <-> ctypes) around the plain C in
``sparcml_oracle.c``; every piece of the method's arithmetic lives there, with
its PAPER.md citation.  ``build()`` compiles it with gcc.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sparcml_oracle.c")
_HDR = os.path.join(_HERE, "sparcml_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB64 = os.path.join(_HERE, "liboracle_f64.so")   # same source, or_val = double

ALGO_AUTO, ALGO_SSAR_RD, ALGO_SSAR_SPLIT, ALGO_DSAR_SPLIT = 0, 1, 2, 3


def build(force: bool = False, f64: bool = False) -> str:
    """Compile oracle/liboracle.so and liboracle_f64.so (gcc, -O2, no FP
    contraction); returns the path of the one asked for."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    for path, extra in ((_LIB, []), (_LIB64, ["-DOR_VAL=double"])):
        if force or not os.path.exists(path) or os.path.getmtime(path) < newest:
            cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                   "-fPIC", "-shared", "-Wall", *extra, "-o", path, _SRC, "-lm"]
            subprocess.run(cmd, check=True)
    return _LIB64 if f64 else _LIB


class _RankStats(C.Structure):
    _fields_ = [("bytes_sent", C.c_uint64), ("bytes_recv", C.c_uint64),
                ("msgs_sent", C.c_uint64), ("pairs_sent", C.c_uint64),
                ("stage_nnz", C.c_uint64 * 8), ("stage_dense", C.c_int * 8)]


_libs = {}


def lib(f64: bool = False):
    """The fp32 build, or (f64=True) the build whose collective simulators use double values."""
    key = bool(f64)
    if key not in _libs:
        _lib = C.CDLL(build(f64=key))
        _libs[key] = _lib
        u64, i32, f32, f64 = C.c_uint64, C.c_int, C.c_float, C.c_double
        p = C.c_void_p
        _lib.or_val_bytes.restype = i32
        _lib.or_val_bytes.argtypes = []
        _lib.or_switch_threshold.restype = u64
        _lib.or_switch_threshold.argtypes = [u64, i32, i32, f64]
        _lib.or_merge_sum.restype = u64
        _lib.or_merge_sum.argtypes = [p, p, u64, p, p, u64, p, p]
        _lib.or_stream_sum.restype = u64
        _lib.or_stream_sum.argtypes = [u64, u64, i32, p, p, u64, i32, p, p, u64, p, p, p]
        _lib.or_brute_force.restype = u64
        _lib.or_brute_force.argtypes = [i32, u64, p, p, p, p, p, p, p]
        _lib.or_ssar_recursive_double.restype = i32
        _lib.or_ssar_recursive_double.argtypes = [i32, u64, u64, p, p, p, i32, p, p, p, p, p]
        _lib.or_split_allgather.restype = i32
        _lib.or_split_allgather.argtypes = [i32, u64, u64, i32, i32, C.c_uint32, u64,
                                            p, p, p, i32, p, p, p, p, p, p]
        _lib.or_sparse_allgather.restype = i32
        _lib.or_sparse_allgather.argtypes = [i32, u64, u64, p, p, p, i32, p, p, p, p, p]
        _lib.or_set_qsgd_norm.restype = i32
        _lib.or_set_qsgd_norm.argtypes = [i32]
        _lib.or_set_op.restype = i32
        _lib.or_set_op.argtypes = [i32]
        _lib.or_brute_force_op.restype = u64
        _lib.or_brute_force_op.argtypes = [i32, u64, p, p, p, p, p]
        _lib.or_apply_update.restype = i32
        _lib.or_apply_update.argtypes = [p, u64, i32, u64, p, p]
        _lib.or_topk.restype = u64
        _lib.or_topk.argtypes = [p, u64, u64, p, p, p]
        _lib.or_ef_topk.restype = u64
        _lib.or_ef_topk.argtypes = [p, p, f32, u64, u64, p, p]
        _lib.or_topk_bucketed.restype = u64
        _lib.or_topk_bucketed.argtypes = [p, u64, u64, u64, p, p, p]
        _lib.or_ef_topk_bucketed.restype = u64
        _lib.or_ef_topk_bucketed.argtypes = [p, p, f32, u64, u64, u64, p, p]
        _lib.or_philox4x32_10.restype = None
        _lib.or_philox4x32_10.argtypes = [p, p, p]
        _lib.or_qsgd_uniform.restype = f32
        _lib.or_qsgd_uniform.argtypes = [u64, u64]
        _lib.or_qsgd_quantize.restype = i32
        _lib.or_qsgd_quantize.argtypes = [p, u64, i32, C.c_uint32, u64, u64, p, p]
        _lib.or_qsgd_dequantize.restype = i32
        _lib.or_qsgd_dequantize.argtypes = [p, p, u64, i32, C.c_uint32, p]
        _lib.or_expected_nnz.restype = f64
        _lib.or_expected_nnz.argtypes = [u64, u64, i32]
    return _libs[key]


def _is64(dtype) -> bool:
    dt = np.dtype(dtype)
    if dt not in (np.float32, np.float64):
        raise ValueError("value dtype must be float32 or float64")
    return dt == np.float64


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _fv(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------
# thin wrappers
# --------------------------------------------------------------------------

def switch_threshold(N, isize=4, c=4, scale=1.0) -> int:
    return int(lib().or_switch_threshold(N, isize, c, scale))


def merge_sum(ia, va, ib, vb, dtype=np.float32):
    ia, va, ib, vb = _u32(ia), _fv(va, dtype), _u32(ib), _fv(vb, dtype)
    n = len(ia) + len(ib)
    io = np.zeros(max(n, 1), np.uint32)
    vo = np.zeros(max(n, 1), dtype)
    m = lib(_is64(dtype)).or_merge_sum(_ptr(ia), _ptr(va), len(ia), _ptr(ib), _ptr(vb), len(ib), _ptr(io), _ptr(vo))
    return io[:m], vo[:m]


def stream_sum(N, delta, a, b, dtype=np.float32):
    """a, b: (dense: bool, idx|None, val).  Returns (dense, idx|None, val)."""
    ad, ai, av = a
    bd, bi, bv = b
    ai = _u32(ai if ai is not None else np.zeros(0)); bi = _u32(bi if bi is not None else np.zeros(0))
    av, bv = _fv(av, dtype), _fv(bv, dtype)
    na = N if ad else len(ai)
    nb = N if bd else len(bi)
    cap = max(na + nb, N, 1)
    oi = np.zeros(cap, np.uint32)
    ov = np.zeros(cap, dtype)
    od = C.c_int(0)
    n = lib(_is64(dtype)).or_stream_sum(N, delta, int(ad), _ptr(ai), _ptr(av), na, int(bd), _ptr(bi), _ptr(bv), nb,
                            C.byref(od), _ptr(oi), _ptr(ov))
    if od.value:
        return True, None, ov[:N].copy()
    return False, oi[:n].copy(), ov[:n].copy()


def _flatten(streams, dtype=np.float32):
    P = len(streams)
    off = np.zeros(P + 1, np.uint64)
    for i, (ii, _) in enumerate(streams):
        off[i + 1] = off[i] + len(ii)
    idx = _u32(np.concatenate([s[0] for s in streams]) if P else np.zeros(0))
    val = _fv(np.concatenate([s[1] for s in streams]) if P else np.zeros(0), dtype)
    if len(idx) == 0:
        idx, val = np.zeros(1, np.uint32), np.zeros(1, dtype)
    return idx, val, off


OP_SUM, OP_MAX, OP_MIN = 0, 1, 2


class op_scope:
    """`with op_scope(OP_MAX): ...` runs the collective simulators with that operator."""

    def __init__(self, op):
        self.op = op

    def __enter__(self):
        for f64 in (False, True):
            if lib(f64).or_set_op(self.op) != 0:
                raise ValueError("unknown operator")
        return self

    def __exit__(self, *exc):
        for f64 in (False, True):
            lib(f64).or_set_op(OP_SUM)


class qsgd_norm_scope:
    """`with qsgd_norm_scope(1): ...` quantizes with the l2-norm scale (R-31)."""

    def __init__(self, norm):
        self.norm = norm

    def __enter__(self):
        if lib().or_set_qsgd_norm(self.norm) != 0:
            raise ValueError("unknown norm")
        return self

    def __exit__(self, *exc):
        lib().or_set_qsgd_norm(0)


def brute_force_op(N, streams, op, dtype=np.float32):
    """(mask, values) of the definition for operator `op`; neutral element off the union."""
    idx, val, off = _flatten(streams, dtype)
    mask = np.zeros(N, np.uint8)
    f32 = np.zeros(N, dtype)
    with op_scope(op):
        lib(_is64(dtype)).or_brute_force_op(len(streams), N, _ptr(idx), _ptr(val), _ptr(off), _ptr(mask), _ptr(f32))
    return mask, f32


def brute_force(N, streams):
    """Returns dict(mask, d64, f32, abs64, K, idx) — the plain definition."""
    idx, val, off = _flatten(streams)
    mask = np.zeros(N, np.uint8)
    d64 = np.zeros(N, np.float64)
    f32 = np.zeros(N, np.float32)
    a64 = np.zeros(N, np.float64)
    K = lib().or_brute_force(len(streams), N, _ptr(idx), _ptr(val), _ptr(off),
                             _ptr(mask), _ptr(d64), _ptr(f32), _ptr(a64))
    return dict(mask=mask, d64=d64, f32=f32, abs64=a64, K=int(K),
                idx=np.nonzero(mask)[0].astype(np.uint32))


def _stats_list(st):
    out = []
    for s in st:
        out.append(dict(bytes_sent=s.bytes_sent, bytes_recv=s.bytes_recv, msgs_sent=s.msgs_sent,
                        pairs_sent=s.pairs_sent, stage_nnz=list(s.stage_nnz),
                        stage_dense=list(s.stage_dense)))
    return out


def _results(P, N, n_out, dense, n, oi, ov):
    res = []
    for r in range(n_out):
        if dense[r]:
            res.append((True, None, ov[r * N:(r + 1) * N].copy()))
        else:
            m = int(n[r])
            res.append((False, oi[r * N:r * N + m].copy(), ov[r * N:r * N + m].copy()))
    return res


def sparse_allgather(N, streams, delta=None, n_out=None, dtype=np.float32):
    """Sparse allgather of streams with disjoint index ranges (R-27).
    Returns (results, stats); raises ValueError if two ranges overlap."""
    P = len(streams)
    if delta is None:
        delta = switch_threshold(N, isize=np.dtype(dtype).itemsize)
    n_out = P if n_out is None else n_out
    idx, val, off = _flatten(streams, dtype)
    dense = np.zeros(P, np.int32)
    n = np.zeros(P, np.uint64)
    oi = np.zeros(max(n_out * N, 1), np.uint32)
    ov = np.zeros(max(n_out * N, 1), dtype)
    st = (_RankStats * P)()
    rc = lib(_is64(dtype)).or_sparse_allgather(P, N, delta, _ptr(idx), _ptr(val), _ptr(off), n_out, _ptr(dense), _ptr(n),
                                   _ptr(oi), _ptr(ov), st)
    if rc == -2:
        raise ValueError("sparse allgather: index ranges of two ranks overlap")
    if rc != 0:
        raise ValueError("or_sparse_allgather rejected its arguments")
    return _results(P, N, n_out, dense, n, oi, ov), _stats_list(st)


def ssar_recursive_double(N, streams, delta=None, n_out=None, dtype=np.float32):
    """dtype float64: the fp64 build (values "single or double");
    default delta then = floor(N*8/12) (P:488-491 with isize = 8)."""
    P = len(streams)
    if delta is None:
        delta = switch_threshold(N, isize=np.dtype(dtype).itemsize)
    n_out = P if n_out is None else n_out
    idx, val, off = _flatten(streams, dtype)
    dense = np.zeros(P, np.int32)
    n = np.zeros(P, np.uint64)
    oi = np.zeros(max(n_out * N, 1), np.uint32)
    ov = np.zeros(max(n_out * N, 1), dtype)
    st = (_RankStats * P)()
    rc = lib(_is64(dtype)).or_ssar_recursive_double(P, N, delta, _ptr(idx), _ptr(val), _ptr(off), n_out,
                                        _ptr(dense), _ptr(n), _ptr(oi), _ptr(ov), st)
    if rc != 0:
        raise ValueError("or_ssar_recursive_double rejected its arguments")
    return _results(P, N, n_out, dense, n, oi, ov), _stats_list(st)


def split_allgather(N, streams, algo=ALGO_AUTO, delta=None, quant_bits=0, bucket=1024,
                    seed=0, n_out=None, dtype=np.float32):
    P = len(streams)
    if delta is None:
        delta = switch_threshold(N, isize=np.dtype(dtype).itemsize)
    n_out = P if n_out is None else n_out
    idx, val, off = _flatten(streams, dtype)
    dense = np.zeros(P, np.int32)
    n = np.zeros(P, np.uint64)
    oi = np.zeros(max(n_out * N, 1), np.uint32)
    ov = np.zeros(max(n_out * N, 1), dtype)
    st = (_RankStats * P)()
    used = C.c_int(0)
    rc = lib(_is64(dtype)).or_split_allgather(P, N, delta, algo, quant_bits, bucket, seed, _ptr(idx), _ptr(val),
                                  _ptr(off), n_out, _ptr(dense), _ptr(n), _ptr(oi), _ptr(ov), st,
                                  C.byref(used))
    if rc != 0:
        raise ValueError("or_split_allgather rejected its arguments")
    return _results(P, N, n_out, dense, n, oi, ov), _stats_list(st), bool(used.value)


def topk(x, k, residual=False):
    x = _f32(x)
    N = len(x)
    m = min(k, N)
    io = np.zeros(max(m, 1), np.uint32)
    vo = np.zeros(max(m, 1), np.float32)
    res = np.zeros(max(N, 1), np.float32) if residual else None
    got = lib().or_topk(_ptr(x), N, k, _ptr(io), _ptr(vo), _ptr(res) if residual else None)
    assert got == m
    if residual:
        return io[:m], vo[:m], res[:N]
    return io[:m], vo[:m]


def ef_topk(eps, grad, alpha, k):
    eps = _f32(eps).copy()
    grad = _f32(grad)
    N = len(eps)
    m = min(k, N)
    io = np.zeros(max(m, 1), np.uint32)
    vo = np.zeros(max(m, 1), np.float32)
    lib().or_ef_topk(_ptr(eps), _ptr(grad), C.c_float(alpha), N, k, _ptr(io), _ptr(vo))
    return io[:m], vo[:m], eps


def bucketed_count(N, k, B):
    """sum over buckets of min(k, |bucket|)."""
    full, tail = divmod(N, B)
    return full * min(k, B) + (min(k, tail) if tail else 0)


def topk_bucketed(x, k, B, residual=False):
    x = _f32(x)
    N = len(x)
    m = bucketed_count(N, k, B)
    io = np.zeros(max(m, 1), np.uint32)
    vo = np.zeros(max(m, 1), np.float32)
    res = np.zeros(max(N, 1), np.float32) if residual else None
    got = lib().or_topk_bucketed(_ptr(x), N, k, B, _ptr(io), _ptr(vo), _ptr(res) if residual else None)
    assert got == m
    if residual:
        return io[:m], vo[:m], res[:N]
    return io[:m], vo[:m]


def ef_topk_bucketed(eps, grad, alpha, k, B):
    eps = _f32(eps).copy()
    grad = _f32(grad)
    N = len(eps)
    m = bucketed_count(N, k, B)
    io = np.zeros(max(m, 1), np.uint32)
    vo = np.zeros(max(m, 1), np.float32)
    got = lib().or_ef_topk_bucketed(_ptr(eps), _ptr(grad), C.c_float(alpha), N, k, B, _ptr(io), _ptr(vo))
    assert got == m
    return io[:m], vo[:m], eps


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().or_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def qsgd_uniform(seed, c) -> float:
    return float(lib().or_qsgd_uniform(seed, c))


def quantized_size(n, bits, bucket):
    return (n * bits + 7) // 8, (n + bucket - 1) // bucket


def qsgd_quantize(x, bits, bucket=1024, seed=0, ctr_base=0):
    x = _f32(x)
    n = len(x)
    cb, ns = quantized_size(n, bits, bucket)
    codes = np.zeros(max(cb, 1), np.uint8)
    scales = np.zeros(max(ns, 1), np.float32)
    rc = lib().or_qsgd_quantize(_ptr(x), n, bits, bucket, seed, ctr_base, _ptr(codes), _ptr(scales))
    if rc != 0:
        raise ValueError("bad quantizer arguments")
    return codes[:cb], scales[:ns]


def qsgd_dequantize(codes, scales, n, bits, bucket=1024):
    codes = np.ascontiguousarray(codes, np.uint8)
    scales = _f32(scales)
    out = np.zeros(max(n, 1), np.float32)
    rc = lib().or_qsgd_dequantize(_ptr(codes), _ptr(scales), n, bits, bucket, _ptr(out))
    if rc != 0:
        raise ValueError("bad quantizer arguments")
    return out[:n]


def apply_update(v, res, N, dtype=np.float32):
    """Algorithm 1's v <- v - g with g an allreduce result (dense, idx, val);
    returns the updated copy of v."""
    d, i, g = res
    v = _fv(v, dtype).copy()
    if len(v) != N:
        raise ValueError("v must hold N values")
    gi = _u32(i if not d else np.zeros(0, np.uint32))
    gv = _fv(g, dtype)
    n = N if d else len(gi)
    rc = lib(_is64(dtype)).or_apply_update(_ptr(v), N, 1 if d else 0, n, _ptr(gi), _ptr(gv))
    if rc != 0:
        raise ValueError("index out of range")
    return v


def expected_nnz(k, N, P) -> float:
    return float(lib().or_expected_nnz(k, N, P))


def result_to_dense(res, N, dtype=np.float32):
    """(dense, idx, val) -> (mask, vector of dtype) for comparisons."""
    d, i, v = res
    if d:
        return np.ones(N, np.uint8), np.asarray(v, dtype)
    mask = np.zeros(N, np.uint8)
    vec = np.zeros(N, dtype)
    mask[i] = 1
    vec[i] = v
    return mask, vec
