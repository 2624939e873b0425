"""The C ABI library without a GPU: it loads, exports every function
include/ucudnn.h declares, and maps errors to status codes (no exception
crosses the boundary)."""
import ctypes as C
import os
import re

import pytest

from paper_1804_04806_b200 import UcudnnError, plan_network_file
from paper_1804_04806_b200._lib import LIB_PATH, PROTOTYPES, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "ucudnn.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ucudnn[A-Z]\w*)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    l = C.CDLL(LIB_PATH)
    names = header_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(l, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(header_functions()) <= set(PROTOTYPES)


def test_error_strings_and_version():
    l = lib()
    assert l.ucudnnGetErrorString(9) == b"UCUDNN_STATUS_NOT_SUPPORTED"
    assert l.ucudnnGetErrorString(3) == b"UCUDNN_STATUS_BAD_PARAM"
    assert l.ucudnnGetVersion() == 100


def test_descriptors_need_no_gpu():
    l = lib()
    d = C.c_void_p()
    assert l.ucudnnCreateTensorDescriptor(C.byref(d)) == 0
    assert l.ucudnnSetTensor4dDescriptor(d, 2, 3, 4, 5) == 0
    n, c, h, w = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    assert l.ucudnnGetTensor4dDescriptor(d, C.byref(n), C.byref(c), C.byref(h), C.byref(w)) == 0
    assert (n.value, c.value, h.value, w.value) == (2, 3, 4, 5)
    assert l.ucudnnSetTensor4dDescriptor(d, 0, 3, 4, 5) == 3  # BAD_PARAM
    assert b"must be" in l.ucudnnGetLastError()
    assert l.ucudnnDestroyTensorDescriptor(d) == 0
    cd = C.c_void_p()
    assert l.ucudnnCreateConvolutionDescriptor(C.byref(cd)) == 0
    assert l.ucudnnSetConvolution2dDescriptor(cd, 1, 1, 1, 1, 2, 2) == 9  # dilation unsupported


def test_parse_errors_map_to_bad_param(tmp_path):
    bad = tmp_path / "bad.net"
    bad.write_text("network x\nminibatch 4\nlayer a channels=3 size=8x8 filters=2 kernel=3\n")
    with pytest.raises(UcudnnError) as e:
        plan_network_file(str(bad), 0, None, None, "wr", "all", 100)
    assert e.value.status == 3 and "bad.net:3" in e.value.message


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = lib().ucudnnCreate(C.byref(h))
    assert st == 8  # EXECUTION_FAILED: no CUDA device


def test_benchmark_devices_rejects_bad_arguments_without_gpu():
    """ucudnnSetBenchmarkDevices validates before touching CUDA: a null
    handle, a negative count, or a null list with n > 0 is BAD_PARAM."""
    f = lib().ucudnnSetBenchmarkDevices
    ids = (C.c_int * 2)(0, 1)
    assert f(None, ids, 2) == 3
    assert f(None, None, 1) == 3
    assert f(None, ids, -1) == 3
