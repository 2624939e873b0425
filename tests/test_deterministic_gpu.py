"""Deterministic BackwardFilter mode (ucudnnSetDeterministic): every BF
algorithm's dW is bit-identical across repeated calls on Gaussian data --
where split-K fp32 atomics would otherwise make it order-dependent -- and
stays within the TF32 tolerance of the fp64 oracle (reference_conv.hpp:
141-180); a micro-batched plan in this mode is deterministic too."""
import numpy as np
import pytest
import torch

from paper_1804_04806_b200 import ConvShape, Handle, algorithm_workspace
from tests.oracle_py import conv_ref, inputs_for

pytestmark = pytest.mark.gpu

SHAPES = [ConvShape(16, 192, 13, 13, 384, 3, 3, 1, 1, 1, 1),   # AlexNet conv3 geometry: many split-K units
          ConvShape(16, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1),    # conv2
          ConvShape(16, 3, 63, 63, 64, 11, 11, 2, 2, 4, 4),    # conv1 geometry (patch kernel)
          ConvShape(8, 64, 28, 28, 128, 1, 1, 0, 0, 2, 2)]     # ResNet 1x1 stride-2 shortcut


def _sid(s):
    return f"{s.N}x{s.C}x{s.H}-k{s.K}r{s.R}s{s.sh}"


@pytest.mark.parametrize("s", SHAPES, ids=_sid)
@pytest.mark.parametrize("algo", [0, 3, 5, 6, 8])
def test_backward_filter_bitwise_repeatable(cuda, algo, s):
    ws_bytes, ok = algorithm_workspace(2, s, algo, s.N)
    if not ok or ws_bytes > (4 << 30):
        pytest.skip("infeasible")
    rng = np.random.default_rng(11)
    x, dy = inputs_for(2, s, rng, integer=False)
    tx, tdy = torch.from_numpy(x).float().cuda(), torch.from_numpy(dy).float().cuda()
    h = Handle(deterministic=True)
    ws = torch.empty(max(ws_bytes, 4) // 4 + 1, device=cuda)
    outs = []
    for _ in range(4):
        dw = torch.full((s.K, s.C, s.R, s.S), float("nan"), device=cuda)
        h.backward_filter(s, tx, tdy, dw, algo, ws)
        torch.cuda.synchronize()
        outs.append(dw.cpu())
    for o in outs[1:]:
        assert torch.equal(o, outs[0]), "dW differs between identical deterministic calls"
    ref = conv_ref(2, s, x, dy)
    got = outs[0].double().numpy()
    assert np.linalg.norm(got - ref) <= 3e-3 * np.linalg.norm(ref)
    h.close()


def test_micro_batched_plan_is_deterministic(cuda, tmp_path):
    s = ConvShape(32, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1)
    rng = np.random.default_rng(12)
    x, dy = inputs_for(2, s, rng, integer=False)
    tx, tdy = torch.from_numpy(x).float().cuda(), torch.from_numpy(dy).float().cuda()
    h = Handle(policy="powerOfTwo", deterministic=True)
    h.set_benchmark_iterations(1, 2)
    algo = h.get_algorithm(2, s, 8 << 20)  # tight limit: several micro-batches
    ws = torch.empty(max(h.workspace_size(algo, 2, s), 4) // 4 + 1, device=cuda)
    res = []
    for _ in range(3):
        dw = torch.zeros(s.K, s.C, s.R, s.S, device=cuda)
        h.backward_filter(s, tx, tdy, dw, algo, ws)
        torch.cuda.synchronize()
        res.append(dw.cpu())
    assert all(torch.equal(r, res[0]) for r in res[1:])
    assert len(h.plan(algo)) >= 1
    ref = conv_ref(2, s, x, dy)
    assert np.linalg.norm(res[0].double().numpy() - ref) <= 3e-3 * np.linalg.norm(ref)
    h.close()
