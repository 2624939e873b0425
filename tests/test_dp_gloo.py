"""Data-parallel host logic on CPU with the gloo backend, world_size 2.

Covers what the 8-GPU path relies on besides NCCL itself: batch sharding,
the rank-0 cost table broadcast (so every rank plans from the same rows and
gets the same plan), and the filter-gradient sum -- checked against the
single-process full-batch filter gradient computed by the fp64 oracle
(BackwardFilter is additive over sample groups, reference
test_reference_conv.cpp:151-170).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_04806_b200 import ConvShape, plan_kernels
from paper_1804_04806_b200.network import allreduce_filter_grads, share_cost_table, shard

HEADER = "kernel_hash,op_type,algorithm,micro_batch,time_us,workspace_bytes,feasible"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_covers_batch():
    for world in (1, 2, 3, 8):
        for gb in (1, 7, 256, 2048):
            parts = [shard(gb, world, r) for r in range(world)]
            assert sum(c for _, c in parts) == gb
            assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(world - 1))


def _worker(rank, world, port, tmp, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from tests.oracle_py import conv_ref, rand_int
        # 1. cost table: rank 0 "benchmarks" (writes rows), the others receive it
        csv = os.path.join(tmp, f"table_{rank}.csv")
        if rank == 0:
            rows = [f"{0xab:016x},Forward,0,{b},{10 * b},0,1" for b in (1, 2, 4)] + \
                   [f"{0xab:016x},Forward,3,{b},{3 * b + 1},{100 * b},1" for b in (1, 2, 4)]
            open(csv, "w").write(HEADER + "\n" + "\n".join(rows) + "\n")
        text = share_cost_table(csv)
        assert open(csv).read() == text
        # 2. every rank plans from the shared table -> identical reports
        k = [0, 4, 1, 1, 1, 1, 1, 1, 0, 0, 1, 1]
        from paper_1804_04806_b200 import kernel_hash
        h = kernel_hash(0, ConvShape(4, 1, 1, 1, 1, 1, 1))
        table = text.replace(f"{0xab:016x}", f"{h:016x}")
        report = plan_kernels("dp", [k], ["conv"], table, "wr", "powerOfTwo", 250)
        # 3. data-parallel BackwardFilter: each rank its shard, then the sum
        s = ConvShape(6, 3, 7, 7, 4, 3, 3, 1, 1, 1, 1)
        rng = np.random.default_rng(99)
        x = rand_int(rng, (s.N, s.C, s.H, s.W))
        dy = rand_int(rng, (s.N, s.K, s.OH, s.OW))
        start, cnt = shard(s.N, world, rank)
        local = conv_ref(2, s.with_batch(cnt), x[start:start + cnt], dy[start:start + cnt])
        g = torch.from_numpy(local)
        allreduce_filter_grads([g])
        full = conv_ref(2, s, x, dy)
        out_q.put((rank, report, bool(np.array_equal(g.numpy(), full))))
    finally:
        dist.destroy_process_group()


def test_two_rank_table_broadcast_and_grad_allreduce(tmp_path):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(tmp_path), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == res[1][1], "ranks planned differently from the same table"
    assert "micro-count" in res[0][1]
    assert all(ok for _, _, ok in res), "all-reduced dw != full-batch dw"
