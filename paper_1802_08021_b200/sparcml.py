"""Thin ctypes binding of libsparcml.so (include/sparcml.h).

Argument marshalling only: every step of the method runs in the library's
CUDA kernels.  torch supplies device memory, the current stream and (for
multi-process worlds) the process group used to exchange CUDA-IPC handles.
There is no CPU fallback: if the library is missing, importing this module
raises.

Index tensors are torch.int32 reinterpreted as uint32; values are
torch.float32.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence, List

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPARCML_LIB") or os.path.join(_HERE, "libsparcml.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(nvcc, sm_100a). There is no CPU fallback.")

_lib = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants --
OK, ERR_INVALID_ARG, ERR_UNSORTED, ERR_NONFINITE, ERR_MISMATCH, ERR_CUDA, ERR_OOM, ERR_STATE = 0, 1, 2, 3, 4, 5, 7, 8
ERR_TIMEOUT = 9                 # a peer's flag did not arrive within the comm's timeout
INJECT_SKIP_RANKS, INJECT_PERTURB_SIG = 1, 2   # loopback failure injection (tests)
ALGO_AUTO, SSAR_RECURSIVE_DOUBLE, SSAR_SPLIT_ALLGATHER, DSAR_SPLIT_ALLGATHER = 0, 1, 2, 3
SPARSE_ALLGATHER = 4   # header algo_used of sparcml_sparse_allgather
OP_SUM, OP_MAX, OP_MIN = 0, 1, 2
REPR_SPARSE, REPR_DENSE = 0, 1
HEADER_BYTES = 64
IPC_HANDLE_BYTES = 128          # CUDA IPC handle + workspace descriptor
MAX_RANKS = 16
HEADER_MAGIC = 0x4D435053
HEADER_MAGIC_F64 = 0x44435053   # results of the fp64 calls (double values)

EXPORTED = [
    "sparcml_version", "sparcml_status_string", "sparcml_opts_default", "sparcml_switch_threshold",
    "sparcml_expected_nnz", "sparcml_result_bytes", "sparcml_result_val_offset", "sparcml_comm_create",
    "sparcml_comm_export_handle", "sparcml_comm_connect", "sparcml_comm_create_local", "sparcml_comm_destroy",
    "sparcml_comm_nranks", "sparcml_comm_workspace", "sparcml_comm_rank", "sparcml_last_error", "sparcml_sparse_allreduce",
    "sparcml_sparse_allreduce_local", "sparcml_barrier", "sparcml_read_header", "sparcml_ops_workspace_bytes",
    "sparcml_ops_workspace_init", "sparcml_merge_sum", "sparcml_topk_workspace_bytes", "sparcml_topk_sparsify",
    "sparcml_ef_topk", "sparcml_topk_status", "sparcml_quantized_size", "sparcml_quantize", "sparcml_dequantize",
    "sparcml_kernel_launches", "sparcml_profile_enable", "sparcml_profile_only", "sparcml_profile_reset",
    "sparcml_profile_read", "sparcml_fuse_streams", "sparcml_layer_ranges", "sparcml_sparse_allgather",
    "sparcml_sparse_allgather_local", "sparcml_apply_update", "sparcml_quantize_norm",
    "sparcml_sparse_allreduce_f64", "sparcml_sparse_allreduce_local_f64", "sparcml_result_bytes_f64",
    "sparcml_result_val_offset_f64", "sparcml_sparse_allgather_f64", "sparcml_sparse_allgather_local_f64",
    "sparcml_apply_update_f64", "sparcml_topk_sample_positions", "sparcml_comm_set_timeout", "sparcml_comm_inject",
]


class Opts(C.Structure):
    _fields_ = [("algo", C.c_int), ("switch_scale", C.c_float), ("index_bytes", C.c_int),
                ("quant_bits", C.c_int), ("quant_bucket", C.c_uint32), ("seed", C.c_uint64),
                ("k_sum_hint", C.c_uint64), ("validate", C.c_int), ("quant_norm", C.c_int)]


class Header(C.Structure):
    _fields_ = [("magic", C.c_uint32), ("repr", C.c_uint32), ("nnz", C.c_uint64), ("N", C.c_uint64),
                ("k_sum", C.c_uint64), ("bytes_sent", C.c_uint64), ("bytes_recv", C.c_uint64),
                ("algo_used", C.c_uint32), ("status", C.c_uint32), ("val_offset", C.c_uint64)]


assert C.sizeof(Header) == HEADER_BYTES

_p, _u64, _i32, _f32, _sz = C.c_void_p, C.c_uint64, C.c_int, C.c_float, C.c_size_t
_sig = {
    "sparcml_version": (C.c_char_p, []),
    "sparcml_status_string": (C.c_char_p, [_i32]),
    "sparcml_opts_default": (None, [C.POINTER(Opts)]),
    "sparcml_switch_threshold": (_u64, [_u64, _i32, _i32, _f32]),
    "sparcml_expected_nnz": (C.c_double, [_u64, _u64, _i32]),
    "sparcml_result_bytes": (_sz, [_u64]),
    "sparcml_result_val_offset": (_sz, [_u64]),
    "sparcml_comm_create": (_i32, [C.POINTER(_p), _i32, _i32, _i32, _u64, _u64]),
    "sparcml_comm_export_handle": (_i32, [_p, _p]),
    "sparcml_comm_connect": (_i32, [_p, _p]),
    "sparcml_comm_create_local": (_i32, [C.POINTER(_p), _i32, _i32, _u64, _u64]),
    "sparcml_comm_destroy": (_i32, [_p]),
    "sparcml_comm_nranks": (_i32, [_p]),
    "sparcml_comm_workspace": (_p, [_p, _i32]),
    "sparcml_comm_rank": (_i32, [_p]),
    "sparcml_last_error": (C.c_char_p, [_p]),
    "sparcml_sparse_allreduce": (_i32, [_p, _p, _p, _u64, _u64, _i32, C.POINTER(Opts), _p, _sz, _p]),
    "sparcml_sparse_allreduce_local": (_i32, [_p, _p, _p, _p, _u64, _i32, C.POINTER(Opts), _p, _sz, _p]),
    "sparcml_sparse_allreduce_f64": (_i32, [_p, _p, _p, _u64, _u64, _i32, C.POINTER(Opts), _p, _sz, _p]),
    "sparcml_sparse_allreduce_local_f64": (_i32, [_p, _p, _p, _p, _u64, _i32, C.POINTER(Opts), _p, _sz, _p]),
    "sparcml_result_bytes_f64": (_sz, [_u64]),
    "sparcml_result_val_offset_f64": (_sz, [_u64]),
    "sparcml_read_header": (_i32, [_p, C.POINTER(Header), _p]),
    "sparcml_barrier": (_i32, [_p, _p]),
    "sparcml_ops_workspace_bytes": (_sz, [_u64]),
    "sparcml_ops_workspace_init": (_i32, [_p, _sz, _p]),
    "sparcml_merge_sum": (_i32, [_p, _p, _u64, _p, _p, _u64, _p, _p, _p, _p, _sz, _p]),
    "sparcml_topk_workspace_bytes": (_sz, [_u64, _u64]),
    "sparcml_topk_sample_positions": (_sz, [_u64, _p, _sz]),
    "sparcml_comm_set_timeout": (_i32, [_p, _u64]),
    "sparcml_comm_inject": (_i32, [_p, _i32, _u64]),
    "sparcml_topk_sparsify": (_i32, [_p, _u64, _u64, _u64, _p, _p, _p, _p, _sz, _p]),
    "sparcml_ef_topk": (_i32, [_p, _p, _f32, _u64, _u64, _u64, _p, _p, _p, _sz, _p]),
    "sparcml_topk_status": (_i32, [_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), _p]),
    "sparcml_quantized_size": (_i32, [_u64, _i32, C.c_uint32, C.POINTER(_sz), C.POINTER(_sz)]),
    "sparcml_quantize": (_i32, [_p, _u64, _i32, C.c_uint32, _u64, _u64, _p, _p, _p]),
    "sparcml_dequantize": (_i32, [_p, _p, _u64, _i32, C.c_uint32, _p, _p]),
    "sparcml_fuse_streams": (_i32, [_i32, _p, _p, _p, _p, _p, _p, _p]),
    "sparcml_apply_update": (_i32, [_p, _p, _p]),
    "sparcml_apply_update_f64": (_i32, [_p, _p, _p]),
    "sparcml_quantize_norm": (_i32, [_p, _u64, _i32, C.c_uint32, _i32, _u64, _u64, _p, _p, _p]),
    "sparcml_sparse_allgather": (_i32, [_p, _p, _p, _u64, _u64, C.POINTER(Opts), _p, _sz, _p]),
    "sparcml_sparse_allgather_local": (_i32, [_p, _p, _p, _p, _u64, C.POINTER(Opts), _p, _sz, _p]),
    "sparcml_sparse_allgather_f64": (_i32, [_p, _p, _p, _u64, _u64, C.POINTER(Opts), _p, _sz, _p]),
    "sparcml_sparse_allgather_local_f64": (_i32, [_p, _p, _p, _p, _u64, C.POINTER(Opts), _p, _sz, _p]),
    "sparcml_layer_ranges": (_i32, [_p, _i32, _p, _p, _p]),
    "sparcml_kernel_launches": (_u64, []),
    "sparcml_profile_enable": (None, [_i32]),
    "sparcml_profile_reset": (None, []),
    "sparcml_profile_only": (None, [C.c_char_p]),
    "sparcml_profile_read": (_i32, [C.c_char_p, C.POINTER(_u64), C.POINTER(C.c_double)]),
}
for _name, (_res, _args) in _sig.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class SparcmlError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"sparcml status {status} ({status_string(status)}): {msg}")
        self.status = status


def status_string(s: int) -> str:
    return _lib.sparcml_status_string(s).decode()


def _check(rc: int, comm=None):
    if rc != OK:
        raise SparcmlError(rc, _lib.sparcml_last_error(comm).decode())


def version() -> str:
    return _lib.sparcml_version().decode()


def kernel_launches() -> int:
    return int(_lib.sparcml_kernel_launches())


def profile_enable(on: bool = True):
    _lib.sparcml_profile_enable(int(on))


def profile_only(name: Optional[str]):
    _lib.sparcml_profile_only(None if name is None else name.encode())


def profile_reset():
    _lib.sparcml_profile_reset()


def profile_read(name: str):
    """(launches, total_ms) recorded for kernel class `name` (syncs its events)."""
    n, ms = C.c_uint64(), C.c_double()
    _check(_lib.sparcml_profile_read(name.encode(), C.byref(n), C.byref(ms)))
    return int(n.value), float(ms.value)


PROFILED_KERNELS = ["topk", "topk_all", "topk_bucketed", "split_push", "split_fused", "owner", "owner_dsar", "ag_publish", "ag_gather",
                    "barrier", "merge", "concat", "rd_push", "rd_stage", "p1_prep", "p1_sparse", "quantize",
                    "dequantize"]


def switch_threshold(N: int, isize: int = 4, c: int = 4, scale: float = 1.0) -> int:
    return int(_lib.sparcml_switch_threshold(N, isize, c, scale))


def expected_nnz(k: int, N: int, P: int) -> float:
    return float(_lib.sparcml_expected_nnz(k, N, P))


def result_bytes(N: int, dtype=torch.float32) -> int:
    if dtype == torch.float64:
        return int(_lib.sparcml_result_bytes_f64(N))
    return int(_lib.sparcml_result_bytes(N))


def result_val_offset(N: int, dtype=torch.float32) -> int:
    if dtype == torch.float64:
        return int(_lib.sparcml_result_val_offset_f64(N))
    return int(_lib.sparcml_result_val_offset(N))


def _val_dtype(t: torch.Tensor):
    """float32, or float64 for the fp64 calls (values "single or double")."""
    if t.dtype not in (torch.float32, torch.float64):
        raise ValueError("val must be float32 or float64")
    return t.dtype


def make_opts(algo: int = ALGO_AUTO, switch_scale: float = 1.0, quant_bits: int = 0, quant_bucket: int = 1024,
              seed: int = 0, k_sum_hint: int = 0, validate: bool = False, quant_norm: int = 0) -> Opts:
    o = Opts()
    _lib.sparcml_opts_default(C.byref(o))
    o.algo, o.switch_scale, o.quant_bits, o.quant_bucket = algo, switch_scale, quant_bits, quant_bucket
    o.seed, o.k_sum_hint, o.validate, o.quant_norm = seed, k_sum_hint, int(validate), quant_norm
    return o


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, dtype, name):
    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous CUDA {dtype} tensor")


# ------------------------------------------------------------------ results --
@dataclass
class Result:
    """Decoded allreduce output (views into the `out` buffer)."""
    header: Header
    dense: bool
    idx: Optional[torch.Tensor]   # int32 [nnz] (sparse) or None
    val: torch.Tensor             # float32 (float64 for the fp64 calls) [nnz] or [N]


def new_out(N: int, device=None, dtype=torch.float32) -> torch.Tensor:
    return torch.empty(result_bytes(N, dtype), dtype=torch.uint8, device=device or "cuda")


def payload_views(out: torch.Tensor, N: int, n: int, dtype=torch.float32):
    """(idx int32[n], val[n]) views of out's sparse payload slots: a stream
    written there (e.g. by the top-k) is an in-place allreduce input."""
    vo = result_val_offset(N, dtype)
    w = torch.empty(0, dtype=dtype).element_size()
    idx = out[HEADER_BYTES:HEADER_BYTES + 4 * n].view(torch.int32)
    val = out[vo:vo + w * n].view(dtype)
    return idx, val


def read_result(out: torch.Tensor, stream=None) -> Result:
    """Synchronises `stream`, reads the header and returns views of the payload."""
    h = Header()
    _check(_lib.sparcml_read_header(out.data_ptr(), C.byref(h), _stream(stream)))
    if h.magic not in (HEADER_MAGIC, HEADER_MAGIC_F64):
        raise SparcmlError(ERR_STATE, "output header not written")
    dt, w = (torch.float64, 8) if h.magic == HEADER_MAGIC_F64 else (torch.float32, 4)
    N = int(h.N)
    if h.repr == REPR_DENSE:
        val = out[HEADER_BYTES:HEADER_BYTES + w * N].view(dt)
        return Result(h, True, None, val)
    n = int(h.nnz)
    idx = out[HEADER_BYTES:HEADER_BYTES + 4 * n].view(torch.int32)
    val = out[h.val_offset:h.val_offset + w * n].view(dt)
    return Result(h, False, idx, val)


# -------------------------------------------------------------- communicators --
def exchange_handles(mine: bytes, group=None) -> bytes:
    """All-gather every rank's workspace handle (CUDA IPC handle + layout descriptor,
    IPC_HANDLE_BYTES) over the process group (host-side bootstrap; any backend) and
    return them concatenated in rank order."""
    import torch.distributed as dist
    if len(mine) != IPC_HANDLE_BYTES:
        raise ValueError(f"handle must be {IPC_HANDLE_BYTES} bytes")
    P = dist.get_world_size(group)
    allh = [None] * P
    dist.all_gather_object(allh, mine, group=group)
    if any(h is None or len(h) != IPC_HANDLE_BYTES for h in allh):
        raise SparcmlError(ERR_MISMATCH, "a rank sent a malformed handle")
    return b"".join(allh)


def _outs_bytes(outs) -> int:
    """The byte capacity every out buffer offers (uint8, contiguous, on the device)."""
    for o in outs:
        if o.dtype != torch.uint8 or not o.is_contiguous() or not o.is_cuda:
            raise ValueError("out buffers must be contiguous uint8 CUDA tensors (new_out)")
    return min(int(o.numel()) for o in outs)


class LocalWorld:
    """All P ranks in this process on one GPU (loopback exchanges)."""

    def __init__(self, P: int, max_N: int, max_nnz: int, device: Optional[int] = None):
        dev = torch.cuda.current_device() if device is None else device
        h = C.c_void_p()
        _check(_lib.sparcml_comm_create_local(C.byref(h), P, dev, max_N, max_nnz))
        self._h, self.P, self.max_N, self.max_nnz, self.device = h, P, max_N, max_nnz, dev

    def allreduce(self, streams: Sequence, N: int, outs: Optional[Sequence[torch.Tensor]] = None,
                  opts: Optional[Opts] = None, stream=None, op: int = OP_SUM):
        """streams: P pairs (idx int32 cuda, val float32 or float64 cuda).  Returns the P out buffers."""
        P = self.P
        assert len(streams) == P
        dt = _val_dtype(streams[0][1])
        for i, v in streams:
            _need(i, torch.int32, "idx")
            _need(v, dt, "val")
        if outs is None:
            outs = [new_out(N, i.device, dt) for i, _ in streams]
        ia = (C.c_void_p * P)(*[_ptr(i) for i, _ in streams])
        va = (C.c_void_p * P)(*[_ptr(v) for _, v in streams])
        na = (C.c_uint64 * P)(*[int(i.numel()) for i, _ in streams])
        oa = (C.c_void_p * P)(*[o.data_ptr() for o in outs])
        o = opts if opts is not None else make_opts()
        fn = _lib.sparcml_sparse_allreduce_local_f64 if dt == torch.float64 else _lib.sparcml_sparse_allreduce_local
        _check(fn(self._h, ia, va, na, N, op, C.byref(o), oa, _outs_bytes(outs), _stream(stream)), self._h)
        return list(outs)

    def allgather(self, streams: Sequence, N: int, outs: Optional[Sequence[torch.Tensor]] = None,
                  opts: Optional[Opts] = None, stream=None):
        """Sparse allgather (§7 SCD, reading R-27): streams with disjoint index ranges.
        Returns the P out buffers (all hold the union)."""
        P = self.P
        dt = _val_dtype(streams[0][1])
        for i, v in streams:
            _need(i, torch.int32, "idx")
            _need(v, dt, "val")
        if outs is None:
            outs = [new_out(N, streams[0][0].device, dt) for _ in range(P)]
        ia = (C.c_void_p * P)(*[_ptr(i) for i, _ in streams])
        va = (C.c_void_p * P)(*[_ptr(v) for _, v in streams])
        na = (C.c_uint64 * P)(*[int(i.numel()) for i, _ in streams])
        oa = (C.c_void_p * P)(*[o.data_ptr() for o in outs])
        o = opts if opts is not None else make_opts()
        fn = _lib.sparcml_sparse_allgather_local_f64 if dt == torch.float64 else _lib.sparcml_sparse_allgather_local
        _check(fn(self._h, ia, va, na, N, C.byref(o), oa, _outs_bytes(outs), _stream(stream)), self._h)
        return outs

    def set_timeout(self, ms: int):
        """Flag waits give up after `ms` milliseconds (header status ERR_TIMEOUT); 0 = never."""
        _check(_lib.sparcml_comm_set_timeout(self._h, int(ms)), self._h)

    def inject(self, what: int, value: int):
        """Failure injection (tests): INJECT_SKIP_RANKS mask, INJECT_PERTURB_SIG rank + 1."""
        _check(_lib.sparcml_comm_inject(self._h, int(what), int(value)), self._h)

    def close(self):
        if self._h:
            _lib.sparcml_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def debug_ctrl(self, rank: int, offset: int, nbytes: int, stream=None) -> bytes:
        """Diagnostics: nbytes of rank's control block at `offset` (syncs)."""
        ptr = _lib.sparcml_comm_workspace(self._h, rank)
        out = bytearray()
        for o in range(0, nbytes, HEADER_BYTES):
            h = Header()
            _check(_lib.sparcml_read_header(ptr + offset + o, C.byref(h), _stream(stream)))
            out += bytes(h)
        return bytes(out[:nbytes])


class Comm:
    """One rank per process; peers' workspaces mapped over NVLink (CUDA IPC).
    Handles are exchanged with torch.distributed (any backend)."""

    def __init__(self, max_N: int, max_nnz: int, group=None, device: Optional[int] = None):
        import torch.distributed as dist
        rank = dist.get_rank(group)
        P = dist.get_world_size(group)
        dev = torch.cuda.current_device() if device is None else device
        h = C.c_void_p()
        _check(_lib.sparcml_comm_create(C.byref(h), P, rank, dev, max_N, max_nnz))
        self._h, self.P, self.rank, self.device = h, P, rank, dev
        if P > 1:
            buf = (C.c_uint8 * IPC_HANDLE_BYTES)()
            _check(_lib.sparcml_comm_export_handle(h, buf), h)
            blob = exchange_handles(bytes(buf), group)
            arr = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
            _check(_lib.sparcml_comm_connect(h, arr), h)

    def allreduce(self, idx: torch.Tensor, val: torch.Tensor, N: int, out: Optional[torch.Tensor] = None,
                  opts: Optional[Opts] = None, stream=None, op: int = OP_SUM) -> torch.Tensor:
        _need(idx, torch.int32, "idx")
        dt = _val_dtype(val)
        _need(val, dt, "val")
        if out is None:
            out = new_out(N, idx.device, dt)
        o = opts if opts is not None else make_opts()
        fn = _lib.sparcml_sparse_allreduce_f64 if dt == torch.float64 else _lib.sparcml_sparse_allreduce
        _check(fn(self._h, _ptr(idx), _ptr(val), int(idx.numel()), N, op, C.byref(o), out.data_ptr(),
                  int(out.numel()), _stream(stream)), self._h)
        return out

    def allgather(self, idx: torch.Tensor, val: torch.Tensor, N: int, out: Optional[torch.Tensor] = None,
                  opts: Optional[Opts] = None, stream=None) -> torch.Tensor:
        """Sparse allgather of streams with disjoint index ranges (§7 SCD, reading R-27)."""
        _need(idx, torch.int32, "idx")
        dt = _val_dtype(val)
        _need(val, dt, "val")
        if out is None:
            out = new_out(N, idx.device, dt)
        o = opts if opts is not None else make_opts()
        fn = _lib.sparcml_sparse_allgather_f64 if dt == torch.float64 else _lib.sparcml_sparse_allgather
        _check(fn(self._h, _ptr(idx), _ptr(val), int(idx.numel()), N, C.byref(o), out.data_ptr(), int(out.numel()),
                  _stream(stream)), self._h)
        return out

    def allreduce_async(self, idx: torch.Tensor, val: torch.Tensor, N: int, out: Optional[torch.Tensor] = None,
                        opts: Optional[Opts] = None, stream=None) -> "Request":
        """Non-blocking allreduce ("layer-wise using non-blocking calls"): enqueued on
        `stream` (default: the current stream) after the work already there; returns a Request
        whose event marks completion.  The host never waits."""
        st = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            out = self.allreduce(idx, val, N, out=out, opts=opts, stream=st)
            ev = torch.cuda.Event()
            ev.record(st)
        return Request(out, ev)

    def barrier(self, stream=None):
        """Device-side barrier of all ranks (stream-ordered, over NVLink flags)."""
        _check(_lib.sparcml_barrier(self._h, _stream(stream)), self._h)

    def set_timeout(self, ms: int):
        """Flag waits give up after `ms` milliseconds (header status ERR_TIMEOUT); 0 = never."""
        _check(_lib.sparcml_comm_set_timeout(self._h, int(ms)), self._h)

    def allreduce_host(self, idx_host, val_host, N: int, out_host=None, opts: Optional[Opts] = None, stream=None):
        """End-to-end path through the C ABI with HOST buffers: H2D of the input,
        the collective, D2H of the result payload.  Returns (header, out_host)."""
        dev_idx = idx_host.to(f"cuda:{self.device}", non_blocking=True)
        dev_val = val_host.to(f"cuda:{self.device}", non_blocking=True)
        out = self.allreduce(dev_idx, dev_val, N, opts=opts, stream=stream)
        if out_host is None:
            out_host = torch.empty(out.numel(), dtype=torch.uint8, pin_memory=True)
        out_host.copy_(out, non_blocking=True)
        return out_host

    def close(self):
        if self._h:
            _lib.sparcml_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------ stream ops ----
def merge_sum(ia: torch.Tensor, va: torch.Tensor, ib: torch.Tensor, vb: torch.Tensor, stream=None):
    """Union-merge-with-sum of two sorted sparse streams.  Syncs to read the count."""
    n = ia.numel() + ib.numel()
    dev = ia.device
    io = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    vo = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    wsb = int(_lib.sparcml_ops_workspace_bytes(n))
    ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
    _check(_lib.sparcml_merge_sum(_ptr(ia), _ptr(va), ia.numel(), _ptr(ib), _ptr(vb), ib.numel(), _ptr(io),
                                  _ptr(vo), cnt.data_ptr(), ws.data_ptr(), wsb, _stream(stream)))
    m = int(cnt.item())
    return io[:m], vo[:m]


class TopkWorkspace:
    def __init__(self, N: int, k: int, device=None):
        self.bytes = int(_lib.sparcml_topk_workspace_bytes(N, k))
        self.buf = torch.zeros(self.bytes, dtype=torch.uint8, device=device or "cuda")
        self.N, self.k = N, k

    def status(self, stream=None):
        st, ps = C.c_uint32(), C.c_uint32()
        _check(_lib.sparcml_topk_status(self.buf.data_ptr(), C.byref(st), C.byref(ps), _stream(stream)))
        return int(st.value), int(ps.value)


def topk_sample_positions(N: int):
    """Diagnostics: start positions of the float4 granules the global top-k samples (current device)."""
    import numpy as np
    n = int(_lib.sparcml_topk_sample_positions(N, None, 0))
    buf = np.zeros(max(n, 1), np.uint64)
    _lib.sparcml_topk_sample_positions(N, buf.ctypes.data_as(C.c_void_p), n)
    return buf[:n]


class Request:
    """Handle of a non-blocking allreduce: `wait(stream)` orders `stream` after it (device
    side, no host sync); `result()` synchronises and returns the Result views."""

    def __init__(self, out: torch.Tensor, event):
        self.out, self.event = out, event

    def wait(self, stream=None):
        (stream if stream is not None else torch.cuda.current_stream()).wait_event(self.event)
        return self.out

    def done(self) -> bool:
        return self.event.query()

    def result(self):
        self.event.synchronize()
        return read_result(self.out)


# ---------------------------------------------------------------- tensor fusion
def layer_offsets(dims: Sequence[int]) -> List[int]:
    """Layers laid end to end: offsets [0, N_0, N_0 + N_1, ...] (L + 1 entries)."""
    off = [0]
    for n in dims:
        off.append(off[-1] + int(n))
    return off


def fuse_streams(streams: Sequence, offsets: Sequence[int], stream=None):
    """One sorted stream over sum(N_l) from L per-layer (idx int32, val float32) streams:
    idx + off_l, concatenated in layer order (one kernel)."""
    L = len(streams)
    if L == 0 or len(offsets) < L:
        raise ValueError("need one offset per layer")
    n = [int(i.numel()) for i, _ in streams]
    dev = streams[0][0].device
    tot = sum(n)
    io = torch.empty(max(tot, 1), dtype=torch.int32, device=dev)
    vo = torch.empty(max(tot, 1), dtype=torch.float32, device=dev)
    for i, v in streams:
        _need(i, torch.int32, "idx")
        _need(v, torch.float32, "val")
    ip = (C.c_void_p * L)(*[i.data_ptr() if i.numel() else None for i, _ in streams])
    vp = (C.c_void_p * L)(*[v.data_ptr() if v.numel() else None for _, v in streams])
    nn = (C.c_uint64 * L)(*n)
    oo = (C.c_uint64 * L)(*[int(o) for o in offsets[:L]])
    _check(_lib.sparcml_fuse_streams(L, ip, vp, nn, oo, io.data_ptr(), vo.data_ptr(), _stream(stream)))
    return io[:tot], vo[:tot]


def layer_ranges(out: torch.Tensor, offsets: Sequence[int], stream=None) -> torch.Tensor:
    """Device tensor (L+1,) int64: layer l's payload positions are [r[l], r[l+1])."""
    L = len(offsets) - 1 if len(offsets) > 1 else 1
    r = torch.empty(L + 1, dtype=torch.int64, device=out.device)
    oo = (C.c_uint64 * L)(*[int(o) for o in offsets[:L]])
    _check(_lib.sparcml_layer_ranges(out.data_ptr(), L, oo, r.data_ptr(), _stream(stream)))
    return r


def split_result(out: torch.Tensor, offsets: Sequence[int], stream=None):
    """Per-layer views (global indices) of a fused allreduce result; synchronises."""
    res = read_result(out, stream)
    r = layer_ranges(out, offsets, stream).cpu().tolist()
    L = len(r) - 1
    if res.header.repr == REPR_DENSE:
        return [(None, res.val[r[l]:r[l + 1]]) for l in range(L)]
    return [(res.idx[r[l]:r[l + 1]], res.val[r[l]:r[l + 1]]) for l in range(L)]


def apply_update(v: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """Algorithm 1's update v <- v - g from an allreduce result, on the device."""
    if v.dtype == torch.float64:   # for an _f64 result
        _need(v, torch.float64, "v")
        _check(_lib.sparcml_apply_update_f64(v.data_ptr(), out.data_ptr(), _stream(stream)))
        return v
    _need(v, torch.float32, "v")
    _check(_lib.sparcml_apply_update(v.data_ptr(), out.data_ptr(), _stream(stream)))
    return v


def algorithm1_step(comm, v: torch.Tensor, eps: torch.Tensor, grad: torch.Tensor, alpha: float, k: int,
                    bucket: int = 0, q_bits: int = 0, q_bucket: int = 512, q_seed: int = 0, opts=None,
                    ws=None, out=None, stream=None):
    """One step of Algorithm 1 at this node, all on the device, no host sync:
    acc = eps + alpha*grad; eps <- acc - TopK(acc); g = allreduce(Q(TopK(acc)), SUM); v <- v - g.
    Q (q_bits = 2/4/8) is QSGD on the k selected values, buckets of q_bucket over the
    value array, Philox counter = rank * (k per rank) + position (reading R-29); q_bits = 0: Q = identity.
    `comm` is a Comm (one rank per process).  Returns the allreduce out buffer."""
    N = v.numel()
    idx, val = ef_topk(eps, grad, alpha, k, ws=ws, stream=stream, bucket=bucket)
    if q_bits:
        codes, scales = quantize(val, q_bits, bucket=q_bucket, seed=q_seed, ctr_base=comm.rank * val.numel(),
                                 stream=stream)
        val = dequantize(codes, scales, val.numel(), q_bits, bucket=q_bucket, stream=stream)
    out = comm.allreduce(idx, val, N, out=out, opts=opts, stream=stream)
    apply_update(v, out, stream=stream)
    return out


def topk_count(N: int, k: int, bucket: int = 0) -> int:
    """Entries a top-k call writes: min(k, N) (global) or sum over buckets of min(k, |bucket|)."""
    if bucket == 0:
        return min(k, N)
    full, tail = divmod(N, bucket)
    return full * min(k, bucket) + (min(k, tail) if tail else 0)


def topk_sparsify(x: torch.Tensor, k: int, residual: Optional[torch.Tensor] = None, ws: Optional[TopkWorkspace] = None,
                  idx_out=None, val_out=None, stream=None, bucket: int = 0):
    """Top-k by magnitude, ties to the lower index; returns (idx int32, val float32) sorted by index.
    bucket > 0 (a multiple of 128, <= 1024): k per bucket of `bucket` consecutive values (§7)."""
    _need(x, torch.float32, "x")
    N = x.numel()
    m = topk_count(N, k, bucket)
    if bucket == 0:
        ws = ws or TopkWorkspace(N, k, x.device)
    io = idx_out if idx_out is not None else torch.empty(m, dtype=torch.int32, device=x.device)
    vo = val_out if val_out is not None else torch.empty(m, dtype=torch.float32, device=x.device)
    _check(_lib.sparcml_topk_sparsify(x.data_ptr(), N, k, bucket, io.data_ptr(), vo.data_ptr(), _ptr(residual),
                                      ws.buf.data_ptr() if ws else None, ws.bytes if ws else 0, _stream(stream)))
    return io, vo


def ef_topk(eps: torch.Tensor, grad: torch.Tensor, alpha: float, k: int, ws: Optional[TopkWorkspace] = None,
            idx_out=None, val_out=None, stream=None, bucket: int = 0):
    """Algorithm 1: acc = eps + alpha*grad (one fma), select TopK(acc), eps <- acc - TopK(acc).
    bucket > 0: the §7 per-bucket selection."""
    _need(eps, torch.float32, "eps")
    _need(grad, torch.float32, "grad")
    N = eps.numel()
    m = topk_count(N, k, bucket)
    if bucket == 0:
        ws = ws or TopkWorkspace(N, k, eps.device)
    io = idx_out if idx_out is not None else torch.empty(m, dtype=torch.int32, device=eps.device)
    vo = val_out if val_out is not None else torch.empty(m, dtype=torch.float32, device=eps.device)
    _check(_lib.sparcml_ef_topk(eps.data_ptr(), grad.data_ptr(), alpha, N, k, bucket, io.data_ptr(), vo.data_ptr(),
                                ws.buf.data_ptr() if ws else None, ws.bytes if ws else 0, _stream(stream)))
    return io, vo


def quantized_size(n: int, bits: int, bucket: int = 1024):
    cb, ns = C.c_size_t(), C.c_size_t()
    _check(_lib.sparcml_quantized_size(n, bits, bucket, C.byref(cb), C.byref(ns)))
    return int(cb.value), int(ns.value)


def quantize(x: torch.Tensor, bits: int, bucket: int = 1024, seed: int = 0, ctr_base: int = 0, stream=None,
             norm: int = 0):
    _need(x, torch.float32, "x")
    n = x.numel()
    cb, ns = quantized_size(n, bits, bucket)
    codes = torch.empty(max(cb, 8), dtype=torch.uint8, device=x.device)
    scales = torch.empty(max(ns, 1), dtype=torch.float32, device=x.device)
    _check(_lib.sparcml_quantize_norm(x.data_ptr(), n, bits, bucket, norm, seed, ctr_base, codes.data_ptr(),
                                      scales.data_ptr(), _stream(stream)))
    return codes[:cb], scales[:ns]


def dequantize(codes: torch.Tensor, scales: torch.Tensor, n: int, bits: int, bucket: int = 1024, stream=None):
    out = torch.empty(n, dtype=torch.float32, device=codes.device)
    _check(_lib.sparcml_dequantize(codes.data_ptr(), scales.data_ptr(), n, bits, bucket, out.data_ptr(),
                                   _stream(stream)))
    return out
