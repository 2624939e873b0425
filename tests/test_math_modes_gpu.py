"""FP32-faithful math mode (ucudnnSetMathMode, "3xTF32"): every algorithm,
run as three TF32 passes over hi / lo operand splits, lands at fp32-level
error against the fp64 oracle (reference_conv.hpp:70-180) on Gaussian data,
where the default TF32 mode sits at ~1e-3 (Winograd / FFT, whose tensor
cores multiply transformed operands, are not offered); its workspace grows by the
operand splits, and a planned, micro-batched call in this mode stays
faithful (BackwardFilter accumulating across micro-batches)."""
import numpy as np
import pytest
import torch

from paper_1804_04806_b200 import ConvShape, Handle
from tests.oracle_py import conv_ref, inputs_for, out_shape

pytestmark = pytest.mark.gpu

SHAPES = [ConvShape(4, 64, 13, 13, 96, 3, 3, 1, 1, 1, 1),
          ConvShape(4, 3, 31, 31, 32, 11, 11, 2, 2, 4, 4),
          ConvShape(4, 32, 14, 14, 64, 1, 1, 0, 0, 2, 2)]
TOL = {}


def _sid(s):
    return f"{s.N}x{s.C}x{s.H}-k{s.K}r{s.R}s{s.sh}"


def _run(h, op, s, a, b, algo):
    import ctypes as C
    from paper_1804_04806_b200._lib import lib
    n = C.c_size_t()
    d = h._d(s)
    st = lib().ucudnnGetConvolutionWorkspaceSize(h._h, algo, op, d.x, d.w, d.c, C.byref(n))
    if st != 0:
        return None, 0
    ws = torch.empty(max(int(n.value), 4) // 4 + 1, device="cuda")
    out = torch.zeros(out_shape(op, s), device="cuda")
    h.run(op, s, torch.from_numpy(a).float().cuda(), torch.from_numpy(b).float().cuda(), out, algo, ws)
    torch.cuda.synchronize()
    return out.cpu().double().numpy(), int(n.value)


@pytest.mark.parametrize("s", SHAPES, ids=_sid)
@pytest.mark.parametrize("op", [0, 1, 2], ids=["F", "BD", "BF"])
@pytest.mark.parametrize("algo", range(9))
def test_fp32_faithful_error(cuda, algo, op, s):
    rng = np.random.default_rng(21 + op)
    a, b = inputs_for(op, s, rng, integer=False)
    ref = conv_ref(op, s, a, b)
    tf32, ws_t = _run(Handle(), op, s, a, b, algo)
    if tf32 is None:
        pytest.skip("infeasible")
    fp32, ws_f = _run(Handle(math="fp32"), op, s, a, b, algo)
    if algo in (1, 2, 4):
        # Winograd / FFT multiply transforms of the operands, which the split
        # cannot make TF32-exact: not offered in this mode
        assert fp32 is None
        return
    e_t = np.linalg.norm(tf32 - ref) / np.linalg.norm(ref)
    e_f = np.linalg.norm(fp32 - ref) / np.linalg.norm(ref)
    assert e_f <= TOL.get(algo, 5e-6), (e_f, e_t)
    assert e_f < e_t / 20 or e_t < 1e-5
    assert ws_f > ws_t


def test_fp32_faithful_planned_backward_filter(cuda):
    s = ConvShape(16, 64, 13, 13, 96, 3, 3, 1, 1, 1, 1)
    rng = np.random.default_rng(5)
    x, dy = inputs_for(2, s, rng, integer=False)
    h = Handle(policy="powerOfTwo", math="fp32")
    h.set_benchmark_iterations(1, 2)
    algo = h.get_algorithm(2, s, 2 << 20)
    ws = torch.empty(max(h.workspace_size(algo, 2, s), 4) // 4 + 1, device=cuda)
    dw = torch.zeros(s.K, s.C, s.R, s.S, device=cuda)
    h.backward_filter(s, torch.from_numpy(x).float().cuda(), torch.from_numpy(dy).float().cuda(), dw, algo, ws)
    torch.cuda.synchronize()
    ref = conv_ref(2, s, x, dy)
    assert np.linalg.norm(dw.cpu().double().numpy() - ref) <= 5e-6 * np.linalg.norm(ref)
