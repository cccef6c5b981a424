"""The C-ABI boundary (include/sparcml.h) without a GPU: the library loads,
exports every function the header declares (and nothing undeclared), and its
host-only utilities agree with the paper's formulas.  No kernel is launched."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sparcml.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(sparcml_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_1802_08021_b200 import build
    path = build.build()
    return path


def test_header_declares_the_hot_path_calls():
    names = declared_functions()
    for must in ["sparcml_sparse_allreduce", "sparcml_topk_sparsify", "sparcml_ef_topk",
                 "sparcml_quantize", "sparcml_dequantize", "sparcml_merge_sum"]:
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = sorted(set(re.findall(r" T (sparcml_[a-z0-9_]+)", out)))
    assert exported == declared_functions()
    h = ctypes.CDLL(lib)
    for n in declared_functions():
        assert hasattr(h, n)


def test_binding_lists_match(lib):
    from paper_1802_08021_b200 import sparcml
    assert sorted(sparcml.EXPORTED) == declared_functions()


def test_host_utilities(lib):
    from paper_1802_08021_b200 import sparcml as S
    assert S.switch_threshold(1024, 4, 4) == 512
    assert S.switch_threshold(8, 8, 4) == 5
    assert S.switch_threshold(1, 4, 4) == 0
    for N in [1, 2, 7, 4096, 2 ** 24, 25_557_032]:
        rb = S.result_bytes(N)
        vo = S.result_val_offset(N)
        H = ((N // 2) + 3) // 4 * 4
        assert vo == 64 + 4 * H
        assert rb >= 64 + 4 * N and rb >= vo + 4 * H
    assert abs(S.expected_nnz(64, 4096, 4) - 250.062255859375) < 1e-6
    assert S.expected_nnz(5, 5, 3) == 5.0
    assert S.status_string(S.ERR_UNSORTED).startswith("input indices")
    assert "sm_100a" in S.version()
    assert S.quantized_size(1000, 4, 1024) == (500, 1)
    assert S.quantized_size(1025, 2, 1024) == (257, 2)


def test_argument_errors_need_no_gpu(lib):
    """Argument validation returns before anything touches the device."""
    from paper_1802_08021_b200 import sparcml as S
    with pytest.raises(S.SparcmlError) as e:
        S._check(S._lib.sparcml_quantized_size(10, 3, 1024, ctypes.byref(ctypes.c_size_t()),
                                               ctypes.byref(ctypes.c_size_t())))
    assert e.value.status == S.ERR_INVALID_ARG
    rc = S._lib.sparcml_topk_sparsify(None, 0, 1, 0, None, None, None, None, 0, None)
    assert rc == S.ERR_INVALID_ARG
    rc = S._lib.sparcml_topk_sparsify(None, 100, 5, 500, None, None, None, None, 0, None)
    assert rc == S.ERR_INVALID_ARG        # bucket must be a multiple of 128
    rc = S._lib.sparcml_topk_sparsify(None, 100, 5, 2048, None, None, None, None, 0, None)
    assert rc == S.ERR_INVALID_ARG        # ... at most 1024
    rc = S._lib.sparcml_topk_sparsify(None, 100, 5, 512, None, None, None, None, 0, None)
    assert rc == S.ERR_INVALID_ARG        # null x
    assert S.topk_count(1000, 4, 512) == 8 and S.topk_count(1100, 600, 512) == 512 + 512 + 76
    assert S.topk_count(10, 3, 0) == 3
    # tensor fusion: argument errors return before any launch
    assert S._lib.sparcml_fuse_streams(0, None, None, None, None, None, None, None) == S.ERR_INVALID_ARG
    two = (ctypes.c_uint64 * 2)
    ptrs = (ctypes.c_void_p * 2)(None, None)
    rc = S._lib.sparcml_fuse_streams(2, ptrs, ptrs, two(0, 0), two(10, 5), None, None, None)
    assert rc == S.ERR_INVALID_ARG        # decreasing layer offsets
    rc = S._lib.sparcml_fuse_streams(2, ptrs, ptrs, two(3, 0), two(0, 5), None, None, None)
    assert rc == S.ERR_INVALID_ARG        # null layer stream with a positive count
    assert S._lib.sparcml_layer_ranges(None, 1, two(0, 0), None, None) == S.ERR_INVALID_ARG
    assert S.layer_offsets([3, 0, 7]) == [0, 3, 3, 10]
    rc = S._lib.sparcml_sparse_allreduce(None, None, None, 0, 10, 0, None, None, 0, None)
    assert rc == S.ERR_INVALID_ARG
