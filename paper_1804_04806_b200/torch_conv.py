"""Framework caller: a PyTorch convolution layer
whose forward and backward run through the C ABI's planned calls.

This is how a framework adopts the library: it keeps
calling the cuDNN-shaped API with a UcudnnHandle_t; Get*Algorithm is called
once per layer shape ("the deep learning framework calls
cudnnGetConvolution*Algorithm one time for each layer prior to the
computation") and returns a virtual algorithm id whose plan the library runs
micro-batch by micro-batch; the framework supplies the workspace from its own
allocator (here torch's caching allocator), as it does for cuDNN.

* `UcudnnConv2d(in_channels, out_channels, kernel_size, stride, padding)`:
  an nn.Module with a KCRS fp32 weight, no bias (the library replaces the
  convolution only; a bias add stays the framework's).
* `conv2d(x, weight, stride, padding, handle)`: the functional form.
* backward computes dx with BackwardData (when x needs a gradient) and dW
  with BackwardFilter (beta = 0: the reference's conv_backward_filter,
  reference_conv.hpp:173-180; torch accumulates into .grad itself).

Tensors are validated before any pointer crosses the ABI: CUDA, float32,
contiguous NCHW, on the handle's device, with the element count the
descriptors imply -- a wrong tensor raises UcudnnError(BAD_PARAM) instead of
becoming an out-of-bounds device access.
"""
from __future__ import annotations

from typing import Dict, Optional, Tuple, Union

import torch

from .api import BACKWARD_DATA, BACKWARD_FILTER, FORWARD, ConvShape, Handle

MiB = 1 << 20
_Pair = Union[int, Tuple[int, int]]


def _pair(v: _Pair) -> Tuple[int, int]:
    return (v, v) if isinstance(v, int) else (int(v[0]), int(v[1]))


class LayerPlans:
    """Virtual algorithm ids of one layer per input shape, queried once each
    (Get*Algorithm for Forward, BackwardData and BackwardFilter)."""

    def __init__(self, handle: Handle, ws_limit: int):
        self.handle = handle
        self.ws_limit = ws_limit
        self.algos: Dict[ConvShape, Tuple[int, int, int]] = {}

    def get(self, s: ConvShape) -> Tuple[int, int, int]:
        a = self.algos.get(s)
        if a is None:
            a = self.algos[s] = tuple(self.handle.get_algorithm(op, s, self.ws_limit)
                                      for op in (FORWARD, BACKWARD_DATA, BACKWARD_FILTER))
        return a

    def workspace(self, algo: int, op: int, s: ConvShape, device) -> Optional[torch.Tensor]:
        n = self.handle.workspace_size(algo, op, s)
        return torch.empty(n, dtype=torch.uint8, device=device) if n else None


class _ConvFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, plans: LayerPlans, s: ConvShape):
        h = plans.handle
        fa, bda, bfa = plans.get(s)
        h.set_stream(torch.cuda.current_stream(x.device).cuda_stream)
        y = torch.empty(s.N, s.K, s.OH, s.OW, device=x.device, dtype=torch.float32)
        h.forward(s, x, weight, y, fa, plans.workspace(fa, FORWARD, s, x.device))
        ctx.save_for_backward(x, weight)
        ctx.plans, ctx.s = plans, s
        return y

    @staticmethod
    def backward(ctx, dy):
        x, weight = ctx.saved_tensors
        plans, s = ctx.plans, ctx.s
        h = plans.handle
        _, bda, bfa = plans.get(s)
        dy = dy.contiguous()
        h.set_stream(torch.cuda.current_stream(dy.device).cuda_stream)
        dx = dw = None
        if ctx.needs_input_grad[0]:
            dx = torch.empty_like(x)
            h.backward_data(s, weight, dy, dx, bda, plans.workspace(bda, BACKWARD_DATA, s, dy.device))
        if ctx.needs_input_grad[1]:
            dw = torch.empty_like(weight)
            h.backward_filter(s, x, dy, dw, bfa, plans.workspace(bfa, BACKWARD_FILTER, s, dy.device))
        return dx, dw, None, None


def conv2d(x: torch.Tensor, weight: torch.Tensor, stride: _Pair = 1, padding: _Pair = 0,
           plans: Optional[LayerPlans] = None, handle: Optional[Handle] = None,
           ws_limit: int = 64 * MiB) -> torch.Tensor:
    """y = conv(x, weight) (cross-correlation, NCHW / KCRS fp32) through the
    library's planned calls; differentiable in x and weight."""
    if plans is None:
        plans = LayerPlans(handle or Handle(), ws_limit)
    if x.dim() != 4 or weight.dim() != 4:
        from ._lib import UcudnnError
        raise UcudnnError(3, "conv2d expects 4-d NCHW input and KCRS weight")
    sh, sw = _pair(stride)
    ph, pw = _pair(padding)
    n, c, hh, ww = x.shape
    k, c2, r, s_ = weight.shape
    s = ConvShape(int(n), int(c), int(hh), int(ww), int(k), int(r), int(s_), ph, pw, sh, sw)
    return _ConvFunction.apply(x, weight, plans, s)


class UcudnnConv2d(torch.nn.Module):
    """nn.Conv2d-shaped layer (no bias, dilation 1, groups 1) running on the
    library. One handle may be shared by every layer of a model (its cost
    table and plan cache then serve them all, as PAPER.md:474-477 describes)."""

    def __init__(self, in_channels: int, out_channels: int, kernel_size: _Pair, stride: _Pair = 1,
                 padding: _Pair = 0, handle: Optional[Handle] = None, ws_limit: int = 64 * MiB,
                 device=None):
        super().__init__()
        r, s = _pair(kernel_size)
        self.stride, self.padding = _pair(stride), _pair(padding)
        self.weight = torch.nn.Parameter(torch.empty(out_channels, in_channels, r, s, device=device))
        torch.nn.init.kaiming_normal_(self.weight)
        self._handle = handle
        self.ws_limit = ws_limit
        self._plans: Optional[LayerPlans] = None

    def plans(self) -> LayerPlans:
        if self._plans is None:
            self._plans = LayerPlans(self._handle or Handle(), self.ws_limit)
        return self._plans

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return conv2d(x, self.weight, self.stride, self.padding, plans=self.plans())

    def extra_repr(self) -> str:
        k, c, r, s = self.weight.shape
        return f"{c}, {k}, kernel_size=({r}, {s}), stride={self.stride}, padding={self.padding}"
