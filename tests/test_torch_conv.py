"""Framework caller: UcudnnConv2d / conv2d as a
torch autograd op over the C ABI, and the tensor validation in front of it.

GPU: a 3-layer model's training step (forward, loss.backward) through the
library equals the fp64 oracle on integer data (every result exact in TF32
and fp32); Get*Algorithm is queried once per layer shape; tensors the
descriptors do not describe raise BAD_PARAM before reaching the device.
CPU: the validation itself (no GPU needed to reject a CPU tensor).
"""
import numpy as np
import pytest
import torch

from paper_1804_04806_b200 import UcudnnError
from paper_1804_04806_b200.api import validate_tensor


def test_validation_rejects_host_and_wrong_tensors():
    with pytest.raises(UcudnnError) as e:
        validate_tensor(torch.zeros(4), 4, "x")
    assert e.value.status == 3 and "CUDA" in str(e.value)
    with pytest.raises(UcudnnError):
        validate_tensor(np.zeros(4), 4, "x")


@pytest.mark.gpu
def test_three_layer_training_step_matches_oracle(cuda):
    from paper_1804_04806_b200 import Handle
    from paper_1804_04806_b200.torch_conv import UcudnnConv2d
    from tests.oracle_py import conv_ref
    h = Handle(policy="powerOfTwo")
    h.set_benchmark_iterations(1, 2)
    layers = [UcudnnConv2d(3, 16, 5, stride=2, padding=2, handle=h, ws_limit=1 << 20, device=cuda),
              UcudnnConv2d(16, 32, 3, padding=1, handle=h, ws_limit=1 << 20, device=cuda),
              UcudnnConv2d(32, 32, 1, handle=h, ws_limit=1 << 20, device=cuda)]
    gen = torch.Generator(device="cpu").manual_seed(3)
    for L in layers:
        with torch.no_grad():
            L.weight.copy_(torch.randint(-1, 2, L.weight.shape, generator=gen).float())
    x = torch.randint(-2, 3, (6, 3, 19, 19), generator=gen).float().to(cuda).requires_grad_()
    # integer, piecewise-linear model: y3 = conv3(conv2(conv1(x))); loss = sum(y3 * g)
    y1 = layers[0](x)
    y2 = layers[1](y1)
    y3 = layers[2](y2)
    g = torch.randint(-1, 2, y3.shape, generator=gen).float().to(cuda)
    (y3 * g).sum().backward()
    torch.cuda.synchronize()
    # oracle chain in fp64
    from paper_1804_04806_b200 import ConvShape
    shapes = [ConvShape(6, 3, 19, 19, 16, 5, 5, 2, 2, 2, 2), ConvShape(6, 16, 10, 10, 32, 3, 3, 1, 1, 1, 1),
              ConvShape(6, 32, 10, 10, 32, 1, 1, 0, 0, 1, 1)]
    ws = [L.weight.detach().cpu().double().numpy() for L in layers]
    a0 = x.detach().cpu().double().numpy()
    a1 = conv_ref(0, shapes[0], a0, ws[0])
    a2 = conv_ref(0, shapes[1], a1, ws[1])
    a3 = conv_ref(0, shapes[2], a2, ws[2])
    assert np.array_equal(y3.detach().cpu().double().numpy(), a3)
    d3 = g.cpu().double().numpy()
    d2 = conv_ref(1, shapes[2], d3, ws[2])
    d1 = conv_ref(1, shapes[1], d2, ws[1])
    d0 = conv_ref(1, shapes[0], d1, ws[0])
    assert np.array_equal(x.grad.cpu().double().numpy(), d0)
    for L, s, a, d in zip(layers, shapes, (a0, a1, a2), (d1, d2, d3)):
        assert np.array_equal(L.weight.grad.cpu().double().numpy(), conv_ref(2, s, a, d))
    # one Get*Algorithm triple per layer shape, reused by a second step
    n_plans = [len(L.plans().algos) for L in layers]
    layers[2](layers[1](layers[0](x))).sum().backward()
    assert n_plans == [1, 1, 1] == [len(L.plans().algos) for L in layers]


@pytest.mark.gpu
def test_bad_tensors_raise_before_the_device(cuda):
    from paper_1804_04806_b200 import ConvShape, Handle
    h = Handle()
    s = ConvShape(2, 4, 8, 8, 8, 3, 3, 1, 1, 1, 1)
    x = torch.zeros(2, 4, 8, 8, device=cuda)
    w = torch.zeros(8, 4, 3, 3, device=cuda)
    y = torch.zeros(2, 8, 8, 8, device=cuda)
    for bad_x in (x.double(), x[:1], x.transpose(2, 3), x.cpu(), torch.zeros(2, 4, 8, 9, device=cuda)):
        with pytest.raises(UcudnnError) as e:
            h.forward(s, bad_x, w, y, 0)
        assert e.value.status == 3
    with pytest.raises(UcudnnError):
        h.backward_filter(s, x, y, torch.zeros(8, 4, 3, 2, device=cuda), 0)
    h.forward(s, x, w, y, 0)  # the well-formed call still runs
    torch.cuda.synchronize()
