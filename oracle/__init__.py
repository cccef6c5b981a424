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

ALGO_AUTO, ALGO_SSAR_RD, ALGO_SSAR_SPLIT, ALGO_DSAR_SPLIT = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile oracle/liboracle.so (gcc, -O2, no FP contraction)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-Wall", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


class _RankStats(C.Structure):
    _fields_ = [("bytes_sent", C.c_uint64), ("bytes_recv", C.c_uint64),
                ("msgs_sent", C.c_uint64), ("pairs_sent", C.c_uint64),
                ("stage_nnz", C.c_uint64 * 8), ("stage_dense", C.c_int * 8)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        u64, i32, f32, f64 = C.c_uint64, C.c_int, C.c_float, C.c_double
        p = C.c_void_p
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
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# --------------------------------------------------------------------------
# thin wrappers
# --------------------------------------------------------------------------

def switch_threshold(N, isize=4, c=4, scale=1.0) -> int:
    return int(lib().or_switch_threshold(N, isize, c, scale))


def merge_sum(ia, va, ib, vb):
    ia, va, ib, vb = _u32(ia), _f32(va), _u32(ib), _f32(vb)
    n = len(ia) + len(ib)
    io = np.zeros(max(n, 1), np.uint32)
    vo = np.zeros(max(n, 1), np.float32)
    m = lib().or_merge_sum(_ptr(ia), _ptr(va), len(ia), _ptr(ib), _ptr(vb), len(ib), _ptr(io), _ptr(vo))
    return io[:m], vo[:m]


def stream_sum(N, delta, a, b):
    """a, b: (dense: bool, idx|None, val).  Returns (dense, idx|None, val)."""
    ad, ai, av = a
    bd, bi, bv = b
    ai = _u32(ai if ai is not None else np.zeros(0)); bi = _u32(bi if bi is not None else np.zeros(0))
    av, bv = _f32(av), _f32(bv)
    na = N if ad else len(ai)
    nb = N if bd else len(bi)
    cap = max(na + nb, N, 1)
    oi = np.zeros(cap, np.uint32)
    ov = np.zeros(cap, np.float32)
    od = C.c_int(0)
    n = lib().or_stream_sum(N, delta, int(ad), _ptr(ai), _ptr(av), na, int(bd), _ptr(bi), _ptr(bv), nb,
                            C.byref(od), _ptr(oi), _ptr(ov))
    if od.value:
        return True, None, ov[:N].copy()
    return False, oi[:n].copy(), ov[:n].copy()


def _flatten(streams):
    P = len(streams)
    off = np.zeros(P + 1, np.uint64)
    for i, (ii, _) in enumerate(streams):
        off[i + 1] = off[i] + len(ii)
    idx = _u32(np.concatenate([s[0] for s in streams]) if P else np.zeros(0))
    val = _f32(np.concatenate([s[1] for s in streams]) if P else np.zeros(0))
    if len(idx) == 0:
        idx, val = np.zeros(1, np.uint32), np.zeros(1, np.float32)
    return idx, val, off


OP_SUM, OP_MAX, OP_MIN = 0, 1, 2


class op_scope:
    """`with op_scope(OP_MAX): ...` runs the collective simulators with that operator."""

    def __init__(self, op):
        self.op = op

    def __enter__(self):
        if lib().or_set_op(self.op) != 0:
            raise ValueError("unknown operator")
        return self

    def __exit__(self, *exc):
        lib().or_set_op(OP_SUM)


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


def brute_force_op(N, streams, op):
    """(mask, values) of the definition for operator `op`; neutral element off the union."""
    idx, val, off = _flatten(streams)
    mask = np.zeros(N, np.uint8)
    f32 = np.zeros(N, np.float32)
    with op_scope(op):
        lib().or_brute_force_op(len(streams), N, _ptr(idx), _ptr(val), _ptr(off), _ptr(mask), _ptr(f32))
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


def sparse_allgather(N, streams, delta=None, n_out=None):
    """Sparse allgather of streams with disjoint index ranges (R-27).
    Returns (results, stats); raises ValueError if two ranges overlap."""
    P = len(streams)
    if delta is None:
        delta = switch_threshold(N)
    n_out = P if n_out is None else n_out
    idx, val, off = _flatten(streams)
    dense = np.zeros(P, np.int32)
    n = np.zeros(P, np.uint64)
    oi = np.zeros(max(n_out * N, 1), np.uint32)
    ov = np.zeros(max(n_out * N, 1), np.float32)
    st = (_RankStats * P)()
    rc = lib().or_sparse_allgather(P, N, delta, _ptr(idx), _ptr(val), _ptr(off), n_out, _ptr(dense), _ptr(n),
                                   _ptr(oi), _ptr(ov), st)
    if rc == -2:
        raise ValueError("sparse allgather: index ranges of two ranks overlap")
    if rc != 0:
        raise ValueError("or_sparse_allgather rejected its arguments")
    return _results(P, N, n_out, dense, n, oi, ov), _stats_list(st)


def ssar_recursive_double(N, streams, delta=None, n_out=None):
    P = len(streams)
    if delta is None:
        delta = switch_threshold(N)
    n_out = P if n_out is None else n_out
    idx, val, off = _flatten(streams)
    dense = np.zeros(P, np.int32)
    n = np.zeros(P, np.uint64)
    oi = np.zeros(max(n_out * N, 1), np.uint32)
    ov = np.zeros(max(n_out * N, 1), np.float32)
    st = (_RankStats * P)()
    rc = lib().or_ssar_recursive_double(P, N, delta, _ptr(idx), _ptr(val), _ptr(off), n_out,
                                        _ptr(dense), _ptr(n), _ptr(oi), _ptr(ov), st)
    if rc != 0:
        raise ValueError("or_ssar_recursive_double rejected its arguments")
    return _results(P, N, n_out, dense, n, oi, ov), _stats_list(st)


def split_allgather(N, streams, algo=ALGO_AUTO, delta=None, quant_bits=0, bucket=1024,
                    seed=0, n_out=None):
    P = len(streams)
    if delta is None:
        delta = switch_threshold(N)
    n_out = P if n_out is None else n_out
    idx, val, off = _flatten(streams)
    dense = np.zeros(P, np.int32)
    n = np.zeros(P, np.uint64)
    oi = np.zeros(max(n_out * N, 1), np.uint32)
    ov = np.zeros(max(n_out * N, 1), np.float32)
    st = (_RankStats * P)()
    used = C.c_int(0)
    rc = lib().or_split_allgather(P, N, delta, algo, quant_bits, bucket, seed, _ptr(idx), _ptr(val),
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


def expected_nnz(k, N, P) -> float:
    return float(lib().or_expected_nnz(k, N, P))


def result_to_dense(res, N):
    """(dense, idx, val) -> (mask, fp32 vector) for comparisons."""
    d, i, v = res
    if d:
        return np.ones(N, np.uint8), np.asarray(v, np.float32)
    mask = np.zeros(N, np.uint8)
    vec = np.zeros(N, np.float32)
    mask[i] = 1
    vec[i] = v
    return mask, vec
