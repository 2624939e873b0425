"""A network's convolution stack run through the C ABI: the bench / DP driver.

Layers come from a `.net` description (reference network.hpp:52-169 format;
configs/*.net). Each layer owns synthetic fp32 NCHW tensors x, w, dy and the
outputs y, dx, dw. A training step runs Forward over all layers, then
BackwardData + BackwardFilter in reverse layer order -- the 3 kernels per
layer of the reference's expand_kernels (network.hpp:183-212) -- each as a
planned (micro-batched) call on the handle's stream. With a process group,
each layer's dw is all-reduced (NCCL sum) on a side stream right after its
last BackwardFilter micro-batch, overlapping the remaining backward.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import List, Optional

import torch

from .api import BACKWARD_DATA, BACKWARD_FILTER, FORWARD, ConvShape, Handle


@dataclass
class Layer:
    name: str
    shape: ConvShape


def parse_net(path: str, batch: Optional[int] = None):
    """Minimal reader of the .net format (network NAME / minibatch N / layer ...)."""
    name, mb, layers = os.path.splitext(os.path.basename(path))[0], 1, []
    for raw in open(path):
        line = raw.split("#", 1)[0].split()
        if not line:
            continue
        if line[0] == "network":
            name = line[1]
        elif line[0] == "minibatch":
            mb = int(line[1])
        elif line[0] == "layer":
            kv = dict(t.split("=", 1) for t in line[2:])
            h, w = map(int, kv["size"].split("x"))
            r, s = map(int, kv["kernel"].split("x"))
            pad, st = int(kv.get("pad", 0)), int(kv.get("stride", 1))
            layers.append((line[1], int(kv["channels"]), h, w, int(kv["filters"]), r, s, pad, st))
    n = batch or mb
    return name, [Layer(nm, ConvShape(n, c, h, w, k, r, s, p, p, st, st)) for nm, c, h, w, k, r, s, p, st in layers]


def shard(global_batch: int, world: int, rank: int):
    """Contiguous data-parallel shard (start, count) of a global mini-batch."""
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def share_cost_table(csv_path: str, group=None) -> str:
    """Rank 0's benchmarked cost table (the reference CSV format,
    cost_database.hpp:32-45) broadcast to every rank, so all ranks plan from
    the same rows -- and the planner being deterministic, run the same plan.
    `csv_path` is rank 0's table on rank 0 and the rank's own copy (written
    here) elsewhere; ranks must not share one path."""
    import torch.distributed as dist
    payload = [open(csv_path).read() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(payload, src=0, group=group)
    if dist.get_rank(group) != 0:
        with open(csv_path, "w") as f:
            f.write(payload[0])
    return payload[0]


def allreduce_filter_grads(grads, group=None, async_op=False):
    """Sum each layer's filter gradient over the data-parallel ranks (the
    caller applies 1/N, reference SPEC.md:370: BackwardFilter has no 1/N)."""
    import torch.distributed as dist
    works = [dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group, async_op=async_op) for g in grads]
    return works if async_op else None


class ConvStack:
    def __init__(self, net_path: str, batch: int, device, seed: int = 1804):
        self.name, self.layers = parse_net(net_path, batch)
        self.device = device
        g = torch.Generator(device="cpu")
        self.t = []
        for i, L in enumerate(self.layers):
            s = L.shape
            g.manual_seed(seed * 1000 + 10 * i)
            x = torch.randn(s.N, s.C, s.H, s.W, generator=g).to(device)
            g.manual_seed(seed * 1000 + 10 * i + 1)
            w = (torch.randn(s.K, s.C, s.R, s.S, generator=g) * (2.0 / (s.C * s.R * s.S)) ** 0.5).to(device)
            g.manual_seed(seed * 1000 + 10 * i + 2)
            dy = torch.randn(s.N, s.K, s.OH, s.OW, generator=g).to(device)
            self.t.append(dict(x=x, w=w, dy=dy, y=torch.empty_like(dy), dx=torch.empty_like(x),
                               dw=torch.empty_like(w)))
        self.algos = None
        self.ws = None
        self.ws_bf = None  # BackwardFilter workspace when BF runs on a side stream
        self.ws_bf_extra = []  # one more per additional side stream

    def kernels(self):
        """(layer index, op) in the reference's expand order: F, BD, BF per layer."""
        return [(i, op) for i in range(len(self.layers)) for op in (FORWARD, BACKWARD_DATA, BACKWARD_FILTER)]

    def flops(self) -> float:
        return 3.0 * sum(L.shape.flops() for L in self.layers)

    def plan(self, h: Handle, ws_limit: int):
        """Get*Algorithm for every kernel (benchmarks missing cost rows, plans WR)."""
        self.algos = {}
        need = 256
        for i, op in self.kernels():
            a = h.get_algorithm(op, self.layers[i].shape, ws_limit)
            self.algos[(i, op)] = a
            need = max(need, h.workspace_size(a, op, self.layers[i].shape))
        self.ws = torch.empty(need // 4 + 64, dtype=torch.float32, device=self.device)
        self.ws_bf = torch.empty(need // 4 + 64, dtype=torch.float32, device=self.device)
        return self.algos

    def run_kernel(self, h: Handle, i: int, op: int):
        s, t, a = self.layers[i].shape, self.t[i], self.algos[(i, op)]
        if op == FORWARD:
            h.forward(s, t["x"], t["w"], t["y"], a, self.ws)
        elif op == BACKWARD_DATA:
            h.backward_data(s, t["w"], t["dy"], t["dx"], a, self.ws)
        else:
            h.backward_filter(s, t["x"], t["dy"], t["dw"], a, self.ws)

    def step(self, h: Handle, comm=None, comm_stream=None, events=None, on_backward=None, on_dw=None,
             bf_stream=None):
        """One training step of the conv stack. `comm`: torch.distributed group
        (dw all-reduce on `comm_stream`); `events`: optional dict (i, op) ->
        (start, end) CUDA events recorded around each kernel; `on_backward()`
        runs before the first backward kernel is issued and `on_dw(i, stream)`
        after layer i's BackwardFilter was issued on `stream` (hooks for
        overlapping host copies).

        `bf_stream` (concurrent kernels): each BackwardFilter runs
        on this side stream with its own workspace (`ws_bf`), overlapping the
        BackwardData chain. The order honours a real network's data flow:
        BF_i needs dy_i, which BD_{i+1} produces, so BF_i waits for BD_{i+1}
        (the top layer's for the forward pass and the incoming gradient);
        BD_i runs right after BD_{i+1} on the main stream; the step joins the
        side stream at its end."""
        cur = torch.cuda.current_stream(self.device)
        n = len(self.layers)
        pending = []

        def after_bf(i, st):
            if on_dw is not None and comm is None:
                on_dw(i, st)
            if comm is not None:
                ev = torch.cuda.Event()
                ev.record(st)
                comm_stream.wait_event(ev)
                with torch.cuda.stream(comm_stream):
                    pending.append(torch.distributed.all_reduce(self.t[i]["dw"], group=comm, async_op=True))

        def run(i, op, st):
            if events is not None:
                events[(i, op)][0].record(st)
            self.run_kernel(h, i, op)
            if events is not None:
                events[(i, op)][1].record(st)

        for i in range(n):
            run(i, FORWARD, cur)
        if on_backward is not None:
            on_backward()
        if bf_stream is None:
            for i in reversed(range(n)):
                run(i, BACKWARD_DATA, cur)
                run(i, BACKWARD_FILTER, cur)
                after_bf(i, cur)
        else:
            # a list of side streams: BF_i on streams[i % len], each with its
            # own workspace, so a BF whose dy is ready need not queue behind
            # the previous layer's BF
            sides = list(bf_stream) if isinstance(bf_stream, (list, tuple)) else [bf_stream]
            while len(self.ws_bf_extra) < len(sides) - 1:
                self.ws_bf_extra.append(torch.empty_like(self.ws_bf))
            wss = [self.ws_bf] + self.ws_bf_extra
            for i in reversed(range(n)):
                ready = torch.cuda.Event()
                ready.record(cur)  # dy_i is available (forward done / BD_{i+1} done)
                run(i, BACKWARD_DATA, cur)
                side = sides[i % len(sides)]
                side.wait_event(ready)
                h.set_stream(side.cuda_stream)
                ws, self.ws = self.ws, wss[i % len(sides)]
                try:
                    run(i, BACKWARD_FILTER, side)
                finally:
                    self.ws = ws
                    h.set_stream(cur.cuda_stream)
                after_bf(i, side)
            for side in sides:
                cur.wait_stream(side)
        if comm is not None:
            for p in pending:
                p.wait()  # makes the current stream wait for the NCCL work
            cur.wait_stream(comm_stream)
