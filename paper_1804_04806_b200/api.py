"""Python mirror of the C ABI (include/ucudnn.h).

Names follow the reference's vocabulary (kernels, micro-batches, policies,
workspace modes, machine reports). Device tensors are torch CUDA tensors;
torch is only the allocator / stream provider here -- every convolution runs
in libucudnn.so's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

from ._lib import UcudnnError, call_string, check, lib

FORWARD, BACKWARD_DATA, BACKWARD_FILTER = 0, 1, 2
OP_NAMES = {FORWARD: "Forward", BACKWARD_DATA: "BackwardData", BACKWARD_FILTER: "BackwardFilter"}
POLICIES = {"all": 0, "powerOfTwo": 1, "undivided": 2}
MODES = {"wr": 0, "wd": 1}
ALGOS = {0: "IMPLICIT_GEMM", 1: "WINOGRAD", 2: "FFT", 3: "GEMM", 4: "WINOGRAD_4x4", 5: "IMPLICIT_PRECOMP_GEMM",
         6: "IMPLICIT_GATHER_GEMM", 7: "IMPLICIT_PRECOMP_GEMM_SLICED",
         8: "IMPLICIT_PRECOMP_GEMM_NHWC"}
VIRTUAL_ALGO_BASE = 1000


@dataclass(frozen=True)
class ConvShape:
    """One convolution layer at batch N (reference KernelDescriptor fields)."""
    N: int
    C: int
    H: int
    W: int
    K: int
    R: int
    S: int
    ph: int = 0
    pw: int = 0
    sh: int = 1
    sw: int = 1

    @property
    def OH(self) -> int:
        return (self.H + 2 * self.ph - self.R) // self.sh + 1

    @property
    def OW(self) -> int:
        return (self.W + 2 * self.pw - self.S) // self.sw + 1

    def with_batch(self, n: int) -> "ConvShape":
        return ConvShape(n, self.C, self.H, self.W, self.K, self.R, self.S, self.ph, self.pw, self.sh, self.sw)

    def as11(self):
        return (C.c_int64 * 11)(self.N, self.C, self.H, self.W, self.K, self.R, self.S, self.ph, self.pw,
                                self.sh, self.sw)

    def flops(self) -> float:
        return 2.0 * self.N * self.K * self.C * self.R * self.S * self.OH * self.OW


def validate_tensor(t, numel: int, name: str, device: Optional[int] = None) -> None:
    """Reject what would become an out-of-bounds or misread device access
    before its pointer crosses the ABI: a CUDA float32 contiguous tensor (on
    the handle's device) with exactly the element count the descriptors
    imply. Raises UcudnnError(BAD_PARAM), as a descriptor mismatch does."""
    def bad(msg):
        raise UcudnnError(3, f"{name}: {msg}")
    if not hasattr(t, "data_ptr") or not hasattr(t, "is_cuda"):
        bad("not a tensor")
    if not t.is_cuda:
        bad("not a CUDA tensor")
    if device is not None and t.device.index != device:
        bad(f"on cuda:{t.device.index}, the handle is on cuda:{device}")
    if str(t.dtype) != "torch.float32":
        bad(f"dtype {t.dtype}, expected float32")
    if not t.is_contiguous():
        bad("not contiguous (packed NCHW / KCRS expected)")
    if t.numel() != numel:
        bad(f"{t.numel()} elements, the descriptor implies {numel}")


def _s(x: Optional[str]) -> Optional[bytes]:
    return None if x is None else x.encode()


def plan_network_file(network: str, batch: int = 0, cost: Optional[str] = None, cache_csv: Optional[str] = None,
                      mode: str = "wr", policy: str = "all", limit: int = 0, jobs: int = 1,
                      report: str = "machine") -> str:
    """`ubatch optimize` through the C ABI (reference tools/main.cpp:116-155)."""
    l = lib()
    return call_string(l.ucudnnPlanNetworkFile, _s(network), batch, _s(cost), _s(cache_csv), MODES[mode],
                       POLICIES[policy], limit, jobs, 1 if report == "text" else 0)


def plan_kernels(name: str, kernels: Sequence[Sequence[int]], names: Sequence[str], cost_csv: str,
                 mode: str = "wr", policy: str = "all", limit: int = 0, jobs: int = 1) -> str:
    """Plans explicit kernels {op,N,C,H,W,K,R,S,ph,pw,sh,sw} against a CSV cost table."""
    l = lib()
    flat = [int(v) for k in kernels for v in k]
    arr = (C.c_int64 * len(flat))(*flat)
    nm = (C.c_char_p * len(names))(*[n.encode() for n in names])
    return call_string(l.ucudnnPlanKernels, _s(name), arr, nm, len(kernels), cost_csv.encode(), MODES[mode],
                       POLICIES[policy], limit, jobs)


def kernel_hash(op: int, s: ConvShape) -> int:
    arr = (C.c_int64 * 12)(op, s.N, s.C, s.H, s.W, s.K, s.R, s.S, s.ph, s.pw, s.sh, s.sw)
    return int(lib().ucudnnKernelHash(arr))


def canonical_time(text: str) -> str:
    """Exact time parse + canonical render (the cost-table time_us column)."""
    return call_string(lib().ucudnnCanonicalTime, text.encode())


def canonical_cost_table(csv_text: str) -> str:
    """Parse a cost-table CSV and re-emit it sorted / canonical."""
    return call_string(lib().ucudnnCanonicalCostTable, csv_text.encode())


def set_trace(on: bool) -> None:
    """Enable (and clear) the process-wide launch-variant trace."""
    check(lib().ucudnnDebugSetTrace(1 if on else 0))


def take_trace() -> list:
    """Launch-variant lines logged since the last call (then cleared)."""
    return [l for l in call_string(lib().ucudnnDebugGetTrace).splitlines() if l]


def algorithm_workspace(op: int, s: ConvShape, algo: int, micro_batch: int):
    ws, ok = C.c_int64(), C.c_int()
    check(lib().ucudnnAlgorithmWorkspace(op, s.as11(), algo, micro_batch, C.byref(ws), C.byref(ok)))
    return int(ws.value), bool(ok.value)


class _Descs:
    """x / w / conv / y descriptors for one shape (freed with the object)."""

    def __init__(self, s: ConvShape):
        l = lib()
        self.x, self.w, self.c, self.y = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(l.ucudnnCreateTensorDescriptor(C.byref(self.x)))
        check(l.ucudnnCreateTensorDescriptor(C.byref(self.y)))
        check(l.ucudnnCreateFilterDescriptor(C.byref(self.w)))
        check(l.ucudnnCreateConvolutionDescriptor(C.byref(self.c)))
        check(l.ucudnnSetTensor4dDescriptor(self.x, s.N, s.C, s.H, s.W))
        check(l.ucudnnSetFilter4dDescriptor(self.w, s.K, s.C, s.R, s.S))
        check(l.ucudnnSetConvolution2dDescriptor(self.c, s.ph, s.pw, s.sh, s.sw, 1, 1))
        check(l.ucudnnSetTensor4dDescriptor(self.y, s.N, s.K, s.OH, s.OW))

    def __del__(self):
        try:
            l = lib()
            l.ucudnnDestroyTensorDescriptor(self.x)
            l.ucudnnDestroyTensorDescriptor(self.y)
            l.ucudnnDestroyFilterDescriptor(self.w)
            l.ucudnnDestroyConvolutionDescriptor(self.c)
        except Exception:
            pass


class Handle:
    """UcudnnHandle_t: device, stream, plans, cost table, WD arena."""

    def __init__(self, policy: str = "powerOfTwo", mode: str = "wr", total_workspace: int = 0,
                 database: Optional[str] = None, stream=None, deterministic: bool = False,
                 math: str = "tf32"):
        self._l = lib()
        self._h = C.c_void_p()
        check(self._l.ucudnnCreate(C.byref(self._h)))
        import torch
        self.device = torch.cuda.current_device()
        self._descs = {}
        self.set_policy(policy)
        self.set_mode(mode)
        if total_workspace:
            self.set_total_workspace(total_workspace)
        # the mode setters start a fresh (mode-specific) cost table, so they
        # come before the database
        if deterministic:
            self.set_deterministic(True)
        if math != "tf32":
            self.set_math_mode(math)
        if database:
            check(self._l.ucudnnSetCostDatabase(self._h, database.encode()))
        if stream is not None:
            self.set_stream(stream)

    def close(self):
        if self._h:
            self._l.ucudnnDestroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- config
    def set_stream(self, stream) -> None:
        ptr = stream if isinstance(stream, int) else getattr(stream, "cuda_stream", 0)
        check(self._l.ucudnnSetStream(self._h, C.c_void_p(ptr)))

    def set_policy(self, policy: str) -> None:
        check(self._l.ucudnnSetBatchSizePolicy(self._h, POLICIES[policy]))

    def set_mode(self, mode: str) -> None:
        check(self._l.ucudnnSetWorkspaceMode(self._h, MODES[mode]))

    def set_total_workspace(self, nbytes: int) -> None:
        check(self._l.ucudnnSetTotalWorkspaceLimit(self._h, nbytes))

    def set_deterministic(self, on: bool) -> None:
        """Run-to-run bit-identical BackwardFilter (no split-K atomics)."""
        check(self._l.ucudnnSetDeterministic(self._h, 1 if on else 0))

    def set_math_mode(self, math: str) -> None:
        """"tf32" (default) or "fp32" (FP32-faithful: 3xTF32 over operand splits)."""
        check(self._l.ucudnnSetMathMode(self._h, {"tf32": 0, "fp32": 1}[math]))

    def set_benchmark_iterations(self, warmup: int, iters: int) -> None:
        check(self._l.ucudnnSetBenchmarkIterations(self._h, warmup, iters))

    def set_benchmark_devices(self, device_ids: Sequence[int]) -> None:
        """Spread the benchmarker's (algorithm x micro-batch) timings over
        these devices, one host thread each; [] = this
        handle's device and stream only."""
        ids = (C.c_int * max(1, len(device_ids)))(*device_ids)
        check(self._l.ucudnnSetBenchmarkDevices(self._h, ids, len(device_ids)))

    def set_database(self, path: str) -> None:
        check(self._l.ucudnnSetCostDatabase(self._h, path.encode()))

    def flush_database(self) -> None:
        check(self._l.ucudnnFlushCostDatabase(self._h))

    def _d(self, s: ConvShape) -> _Descs:
        d = self._descs.get(s)
        if d is None:
            d = self._descs[s] = _Descs(s)
        return d

    # ---------------------------------------------------------------- planning
    def get_algorithm(self, op: int, s: ConvShape, ws_limit: int) -> int:
        d = self._d(s)
        a = C.c_int()
        if op == FORWARD:
            st = self._l.ucudnnGetConvolutionForwardAlgorithm(self._h, d.x, d.w, d.c, d.y, ws_limit, C.byref(a))
        elif op == BACKWARD_DATA:
            st = self._l.ucudnnGetConvolutionBackwardDataAlgorithm(self._h, d.w, d.y, d.c, d.x, ws_limit,
                                                                   C.byref(a))
        else:
            st = self._l.ucudnnGetConvolutionBackwardFilterAlgorithm(self._h, d.x, d.y, d.c, d.w, ws_limit,
                                                                     C.byref(a))
        check(st)
        return a.value

    def workspace_size(self, algo: int, op: int, s: ConvShape) -> int:
        d = self._d(s)
        n = C.c_size_t()
        check(self._l.ucudnnGetConvolutionWorkspaceSize(self._h, algo, op, d.x, d.w, d.c, C.byref(n)))
        return int(n.value)

    def optimize_network(self) -> None:
        check(self._l.ucudnnOptimizeNetwork(self._h))

    def plan(self, algo: int):
        n = C.c_int()
        algs = (C.c_int * 512)()
        bs = (C.c_int64 * 512)()
        check(self._l.ucudnnGetPlan(self._h, algo, C.byref(n), algs, bs, 512))
        return [(int(algs[i]), int(bs[i])) for i in range(n.value)]

    def machine_report(self) -> str:
        return call_string(self._l.ucudnnGetMachineReport, self._h)

    def time_algorithm(self, op: int, s: ConvShape, algo: int, micro_batch: int):
        t, ws, ok = C.c_double(), C.c_int64(), C.c_int()
        check(self._l.ucudnnTimeAlgorithm(self._h, op, s.as11(), algo, micro_batch, C.byref(t), C.byref(ws),
                                          C.byref(ok)))
        return float(t.value), int(ws.value), bool(ok.value)

    def benchmark_kernel(self, op: int, s: ConvShape, policy: str) -> None:
        check(self._l.ucudnnBenchmarkKernel(self._h, op, s.as11(), POLICIES[policy]))

    # ---------------------------------------------------------------- execution
    def _ws(self, ws):
        if ws is None:
            return None, 0
        if not getattr(ws, "is_cuda", False) or not ws.is_contiguous() or ws.device.index != self.device:
            raise UcudnnError(3, "workspace: must be a contiguous CUDA tensor on the handle's device")
        return C.c_void_p(ws.data_ptr()), ws.numel() * ws.element_size()

    def _check(self, s: ConvShape, op: int, a, b, out):
        x_n, w_n, y_n = s.N * s.C * s.H * s.W, s.K * s.C * s.R * s.S, s.N * s.K * s.OH * s.OW
        names = [("x", "w", "y"), ("dy", "w", "dx"), ("x", "dy", "dw")][op]
        sizes = [(x_n, w_n, y_n), (y_n, w_n, x_n), (x_n, y_n, w_n)][op]
        for t, n, nm in zip((a, b, out), sizes, names):
            validate_tensor(t, n, nm, self.device)

    def forward(self, s: ConvShape, x, w, y, algo: int, ws=None, alpha: float = 1.0, beta: float = 0.0):
        self._check(s, FORWARD, x, w, y)
        d = self._d(s)
        wp, wn = self._ws(ws)
        a, b = C.c_float(alpha), C.c_float(beta)
        check(self._l.ucudnnConvolutionForward(self._h, C.byref(a), d.x, C.c_void_p(x.data_ptr()), d.w,
                                               C.c_void_p(w.data_ptr()), d.c, algo, wp, wn, C.byref(b), d.y,
                                               C.c_void_p(y.data_ptr())))

    def backward_data(self, s: ConvShape, w, dy, dx, algo: int, ws=None, alpha: float = 1.0, beta: float = 0.0):
        self._check(s, BACKWARD_DATA, dy, w, dx)
        d = self._d(s)
        wp, wn = self._ws(ws)
        a, b = C.c_float(alpha), C.c_float(beta)
        check(self._l.ucudnnConvolutionBackwardData(self._h, C.byref(a), d.w, C.c_void_p(w.data_ptr()), d.y,
                                                    C.c_void_p(dy.data_ptr()), d.c, algo, wp, wn, C.byref(b),
                                                    d.x, C.c_void_p(dx.data_ptr())))

    def backward_filter(self, s: ConvShape, x, dy, dw, algo: int, ws=None, alpha: float = 1.0,
                        beta: float = 0.0):
        self._check(s, BACKWARD_FILTER, x, dy, dw)
        d = self._d(s)
        wp, wn = self._ws(ws)
        a, b = C.c_float(alpha), C.c_float(beta)
        check(self._l.ucudnnConvolutionBackwardFilter(self._h, C.byref(a), d.x, C.c_void_p(x.data_ptr()), d.y,
                                                      C.c_void_p(dy.data_ptr()), d.c, algo, wp, wn, C.byref(b),
                                                      d.w, C.c_void_p(dw.data_ptr())))

    def run(self, op: int, s: ConvShape, a, b, out, algo: int, ws=None, alpha: float = 1.0, beta: float = 0.0):
        """Uniform entry: op 0 (x, w -> y), 1 (dy, w -> dx), 2 (x, dy -> dw)."""
        if op == FORWARD:
            self.forward(s, a, b, out, algo, ws, alpha, beta)
        elif op == BACKWARD_DATA:
            self.backward_data(s, b, a, out, algo, ws, alpha, beta)
        else:
            self.backward_filter(s, a, b, out, algo, ws, alpha, beta)
