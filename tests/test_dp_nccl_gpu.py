"""The data-parallel step path (SURVEY.md section 8 row e) on the one GPU
this environment has: NCCL at world size 1.

* In-process: ConvStack.step(comm=...) with an NCCL process group, the dW
  all-reduce issued per layer on a side stream after that layer's last
  BackwardFilter micro-batch, BackwardFilter on side streams -- checked
  against the fp64 oracle on integer data (an all-reduce over one rank is
  the identity, so dW must equal the full-batch oracle exactly).
* As the driver launches it: `torch.distributed.run --nproc-per-node 1
  bench.py --gpus 1` (WORLD_SIZE set => the NCCL path), which must print a
  JSON line with n_gpus 1 and a communicator of size 1.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from tests.oracle_py import conv_ref

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_conv_stack_step_with_nccl_allreduce(cuda, tmp_path):
    import torch.distributed as dist
    from paper_1804_04806_b200 import Handle
    from paper_1804_04806_b200.network import ConvStack
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=cuda)
    try:
        net = tmp_path / "tiny.net"
        net.write_text("network tiny\nminibatch 16\n"
                       "layer c1 channels=3 size=27x27 filters=32 kernel=5x5 pad=2 stride=2\n"
                       "layer c2 channels=32 size=14x14 filters=64 kernel=3x3 pad=1 stride=1\n"
                       "layer c3 channels=64 size=14x14 filters=64 kernel=3x3 pad=1 stride=1\n")
        stack = ConvStack(str(net), 16, cuda)
        gen = torch.Generator(device="cpu").manual_seed(5)
        for t in stack.t:
            for k in ("x", "w", "dy"):
                t[k].copy_(torch.randint(-3, 4, t[k].shape, generator=gen).float())
        # a tight limit so some kernels split into micro-batches
        h = Handle(policy="powerOfTwo", database=str(tmp_path / "db.csv"))
        stack.plan(h, 1 << 20)
        comm_stream = torch.cuda.Stream(cuda)
        sides = [torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)]
        for t in stack.t:
            for k in ("y", "dx", "dw"):
                t[k].fill_(float("nan"))
        stack.step(h, dist.group.WORLD, comm_stream, bf_stream=sides)
        torch.cuda.synchronize()
        for L, t in zip(stack.layers, stack.t):
            s = L.shape
            x, w, dy = (t[k].cpu().double().numpy() for k in ("x", "w", "dy"))
            assert np.array_equal(t["y"].cpu().double().numpy(), conv_ref(0, s, x, w)), L.name
            assert np.array_equal(t["dx"].cpu().double().numpy(), conv_ref(1, s, dy, w)), L.name
            assert np.array_equal(t["dw"].cpu().double().numpy(), conv_ref(2, s, x, dy)), L.name
        h.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["graph", "eager"])
def test_bench_under_torchrun_world1(cuda, mode):
    """Both data-parallel schedules of bench.py as the driver launches them:
    graph replay + one bucketed all-reduce of all dW per step (default), and
    eager launches with per-layer all-reduces on a side stream."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "1", "--steps", "2", "--warmup", "3", "--no-cpu"] + (["--dist-eager"] if mode == "eager" else [])
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["config"]["comm_size"] == 1
    if mode == "eager":
        assert line["config"]["launch"].startswith("eager")
    else:
        assert "bucketed NCCL all-reduce" in line["config"]["launch"]
    assert line["value"] > 0 and line["gpu_launches"] > 0
