"""ctypes binding of include/ucudnn.h (the C ABI in libucudnn.so).

The shared library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_1804_04806_b200/csrc``). Loading fails loudly if it is missing: there is
no Python or CPU fallback for any product path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libucudnn.so")

_lock = threading.Lock()
_lib = None

i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
vp = C.c_void_p

# name -> (restype, argtypes); mirrors include/ucudnn.h exactly.
PROTOTYPES = {
    "ucudnnGetErrorString": (C.c_char_p, [C.c_int]),
    "ucudnnGetLastError": (C.c_char_p, []),
    "ucudnnGetMinTotalWorkspace": (i64, []),
    "ucudnnGetVersion": (C.c_size_t, []),
    "ucudnnGetLaunchCount": (C.c_uint64, []),
    "ucudnnDebugPrecompProfile": (C.c_int, [C.POINTER(C.c_double)]),
    "ucudnnDebugBackwardFilterProfile": (C.c_int, [C.POINTER(C.c_double)]),
    "ucudnnDebugSetTrace": (C.c_int, [C.c_int]),
    "ucudnnDebugGetTrace": (C.c_int, [C.c_char_p, C.POINTER(C.c_size_t)]),
    "ucudnnCreate": (C.c_int, [C.POINTER(vp)]),
    "ucudnnDestroy": (C.c_int, [vp]),
    "ucudnnSetStream": (C.c_int, [vp, vp]),
    "ucudnnGetStream": (C.c_int, [vp, C.POINTER(vp)]),
    "ucudnnSetBatchSizePolicy": (C.c_int, [vp, C.c_int]),
    "ucudnnSetWorkspaceMode": (C.c_int, [vp, C.c_int]),
    "ucudnnSetTotalWorkspaceLimit": (C.c_int, [vp, i64]),
    "ucudnnSetCostDatabase": (C.c_int, [vp, C.c_char_p]),
    "ucudnnFlushCostDatabase": (C.c_int, [vp]),
    "ucudnnSetBenchmarkIterations": (C.c_int, [vp, C.c_int, C.c_int]),
    "ucudnnSetDeterministic": (C.c_int, [vp, C.c_int]),
    "ucudnnSetMathMode": (C.c_int, [vp, C.c_int]),
    "ucudnnSetBenchmarkDevices": (C.c_int, [vp, C.POINTER(C.c_int), C.c_int]),
    "ucudnnCreateTensorDescriptor": (C.c_int, [C.POINTER(vp)]),
    "ucudnnSetTensor4dDescriptor": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int]),
    "ucudnnGetTensor4dDescriptor": (C.c_int, [vp] + [C.POINTER(C.c_int)] * 4),
    "ucudnnDestroyTensorDescriptor": (C.c_int, [vp]),
    "ucudnnCreateFilterDescriptor": (C.c_int, [C.POINTER(vp)]),
    "ucudnnSetFilter4dDescriptor": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int]),
    "ucudnnDestroyFilterDescriptor": (C.c_int, [vp]),
    "ucudnnCreateConvolutionDescriptor": (C.c_int, [C.POINTER(vp)]),
    "ucudnnSetConvolution2dDescriptor": (C.c_int, [vp] + [C.c_int] * 6),
    "ucudnnGetConvolution2dForwardOutputDim": (C.c_int, [vp, vp, vp] + [C.POINTER(C.c_int)] * 4),
    "ucudnnDestroyConvolutionDescriptor": (C.c_int, [vp]),
    "ucudnnGetConvolutionForwardAlgorithm": (C.c_int, [vp, vp, vp, vp, vp, i64, C.POINTER(C.c_int)]),
    "ucudnnGetConvolutionBackwardDataAlgorithm": (C.c_int, [vp, vp, vp, vp, vp, i64, C.POINTER(C.c_int)]),
    "ucudnnGetConvolutionBackwardFilterAlgorithm": (C.c_int, [vp, vp, vp, vp, vp, i64, C.POINTER(C.c_int)]),
    "ucudnnGetConvolutionWorkspaceSize": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, C.POINTER(C.c_size_t)]),
    "ucudnnOptimizeNetwork": (C.c_int, [vp]),
    "ucudnnGetPlan": (C.c_int, [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), i64p, C.c_int]),
    "ucudnnGetMachineReport": (C.c_int, [vp, C.c_char_p, C.POINTER(C.c_size_t)]),
    "ucudnnConvolutionForward": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, C.c_int, vp, C.c_size_t, vp, vp, vp]),
    "ucudnnConvolutionBackwardData": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, C.c_int, vp, C.c_size_t, vp, vp, vp]),
    "ucudnnConvolutionBackwardFilter": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, C.c_int, vp, C.c_size_t, vp, vp, vp]),
    "ucudnnTimeAlgorithm": (C.c_int, [vp, C.c_int, i64p, C.c_int, i64, C.POINTER(C.c_double), i64p,
                                      C.POINTER(C.c_int)]),
    "ucudnnBenchmarkKernel": (C.c_int, [vp, C.c_int, i64p, C.c_int]),
    "ucudnnAlgorithmWorkspace": (C.c_int, [C.c_int, i64p, C.c_int, i64, i64p, C.POINTER(C.c_int)]),
    "ucudnnPlanNetworkFile": (C.c_int, [C.c_char_p, i64, C.c_char_p, C.c_char_p, C.c_int, C.c_int, i64,
                                        C.c_uint, C.c_int, C.c_char_p, C.POINTER(C.c_size_t)]),
    "ucudnnPlanKernels": (C.c_int, [C.c_char_p, i64p, C.POINTER(C.c_char_p), C.c_int, C.c_char_p, C.c_int,
                                    C.c_int, i64, C.c_uint, C.c_char_p, C.POINTER(C.c_size_t)]),
    "ucudnnKernelHash": (C.c_uint64, [i64p]),
    "ucudnnCanonicalTime": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_size_t)]),
    "ucudnnCanonicalCostTable": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_size_t)]),
}

STATUS = {0: "SUCCESS", 1: "NOT_INITIALIZED", 2: "ALLOC_FAILED", 3: "BAD_PARAM", 4: "INTERNAL_ERROR",
          5: "INVALID_VALUE", 6: "ARCH_MISMATCH", 8: "EXECUTION_FAILED", 9: "NOT_SUPPORTED"}


class UcudnnError(RuntimeError):
    def __init__(self, status: int, message: str, min_total_workspace: int = -1):
        super().__init__(f"UCUDNN_STATUS_{STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message
        self.min_total_workspace = min_total_workspace


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                                  "(make -C paper_1804_04806_b200/csrc). There is no fallback.")
            l = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
            for name, (res, args) in PROTOTYPES.items():
                fn = getattr(l, name)
                fn.restype = res
                fn.argtypes = args
            _lib = l
        return _lib


def check(status: int) -> None:
    if status != 0:
        l = lib()
        msg = l.ucudnnGetLastError().decode(errors="replace")
        raise UcudnnError(status, msg, int(l.ucudnnGetMinTotalWorkspace()))


def call_string(fn, *args) -> str:
    """Calls an entry point that fills (char* out, size_t* len); grows the buffer once."""
    n = C.c_size_t(1 << 16)
    for _ in range(2):
        buf = C.create_string_buffer(n.value)
        st = fn(*args, buf, C.byref(n))
        if st == 0:
            return buf.value.decode()
        if st != 3 or n.value <= len(buf):
            check(st)
    check(st)
    return ""
