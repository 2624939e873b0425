#!/usr/bin/env python3
"""Headline benchmark: AlexNet bs256 conv fwd+bwd ms/iter at a 64 MiB
per-kernel workspace limit (WR), and the speedup over the undivided plan
(BASELINE.json `metric`; configs C2 / C5 of SURVEY.md section 8).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One process per GPU (torchrun for N > 1): each rank micro-batches its own
bs256 shard with the same plan and all-reduces every layer's filter gradient
over NCCL (weak scaling). Timing: CUDA events on the compute stream over K
steps after W warm-up steps, barrier + synchronize on both sides, max over
ranks. The step's working set (AlexNet activations ~1.1 GB) exceeds the
126 MB L2, so no explicit flush is needed between steps. Rank 0 prints one
JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MiB = 1 << 20
METRIC = "AlexNet bs256 conv fwd+bwd ms/iter @64 MiB WS; speedup vs undivided"


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


_JSON_FD = None


def quiet_stdout():
    """Route everything written to stdout (NCCL's version banner, library
    prints) to stderr at the file-descriptor level, keeping the real stdout
    for the one JSON line (emit)."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(obj) -> None:
    sys.stdout.flush()
    data = (json.dumps(obj) + "\n").encode()
    if _JSON_FD is None:
        os.write(1, data)
    else:
        os.write(_JSON_FD, data)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this command under
    torch.distributed.run with N ranks (one process per GPU, rendezvous on
    127.0.0.1), exactly as the driver's torchrun launch would."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------ CPU reference arm
def cpu_reference(net_path: str, sample_n: int, threads: int):
    """The reference fp64 convolution (oracle/_ref/ref_conv.so, compiled from
    /root/reference/proj/include/ubatch/reference_conv.hpp) on `sample_n`
    samples of every AlexNet kernel, all host threads; returns (seconds for
    the sample, extrapolated ms per bs256 iteration, kind)."""
    import numpy as np
    from paper_1804_04806_b200.network import parse_net
    from tests import oracle_py
    _, layers = parse_net(net_path, 256)
    rng = np.random.default_rng(0)
    use_ref = oracle_py.ref_available()
    total = 0.0
    for L in layers:
        s = L.shape.with_batch(sample_n)
        for op in range(3):
            a, b = oracle_py.inputs_for(op, s, rng, integer=False)
            t0 = time.perf_counter()
            if use_ref:
                oracle_py.ref_conv_threads(op, s, a, b, threads)
            else:
                oracle_py.oracle().oracle_set_threads(threads)
                oracle_py.conv_ref(op, s, a, b)
            total += time.perf_counter() - t0
    return total, total * 1e3 * 256.0 / sample_n, ("reference" if use_ref else "port")


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    net = os.path.join(ROOT, "configs", "alexnet.net")
    sample_n = args.ref_sample
    for _ in range(args.warmup):
        cpu_reference(net, sample_n, threads)
    vals = []
    for _ in range(args.steps):
        _, ms, kind = cpu_reference(net, sample_n, threads)
        vals.append(ms)
    # the job's global batch is 256 images per GPU: the host runs all of them
    v = statistics.median(vals) * world
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms/iter", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v, 3), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "alexnet conv layers, Forward + BackwardData + BackwardFilter (15 kernels), "
                                   "batch 256 per GPU", "net": "alexnet", "global_batch": 256 * world,
                       "ws_limit_bytes": 64 * MiB, "mode": "wr", "policy": "powerOfTwo",
                       "parallelism": f"dp{world}"},
            "cpu_baseline": {"value": round(v, 3), "unit": "ms/iter", "cores": threads, "kind": kind,
                             "cpu_model": cpu_model(),
                             "sample": f"{sample_n} of 256 samples of all 15 kernels per step, "
                                       f"x{256 // sample_n} (x{world} ranks' shards)" if world > 1 else
                                       f"{sample_n} of 256 samples of all 15 kernels per step, x{256 // sample_n}"},
            "e2e": {"value": round(v, 3), "unit": "ms/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        # nvidia-smi takes a few hundred ms to start: wait for its first row so
        # the samples fall inside the timed region that follows
        t0 = time.time()
        while self.p is not None and time.time() - t0 < 5.0:
            if os.path.getsize(self.f.name) > 0:
                break
            time.sleep(0.02)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows if len(r) >= 9 for j in range(4) if r[5 + j].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------ GPU arm
def timed(fn, steps, warmup, dev, dist_on):
    import torch
    for _ in range(warmup):
        fn()
    if dist_on:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    if dist_on:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
        ms = float(t.item())
    return ms


def dom_traffic(name, plan):
    """DRAM bytes (read + write) of the dominant call, from the committed ncu
    capture of the same planned step (scripts/traffic.py -> profiles/); null
    when that capture's plan for this call differs from this run's."""
    path = os.path.join(ROOT, "profiles", "r01_traffic.json")
    try:
        rec = json.load(open(path))["calls"].get(name)
    except (OSError, ValueError, KeyError):
        return None
    if not rec or rec["plan"] != plan:
        return None
    return rec["dram_bytes"]


def tf32_peak(dev):
    """cuBLAS TF32 GEMM (8192^3, best of 10) -- the tensor-pipe roofline
    denominator for TF32 kernels (MEASURED_PEAKS.json carries bf16 only)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(8192, 8192, device=dev)
    b = torch.randn(8192, 8192, device=dev)
    best = 1e9
    for i in range(13):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            best = min(best, e0.elapsed_time(e1))
    torch.backends.cuda.matmul.allow_tf32 = False
    return 2 * 8192 ** 3 / (best * 1e-3) / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--net", default="alexnet")
    ap.add_argument("--policy", default="powerOfTwo")
    ap.add_argument("--limit-mib", type=int, default=64, help="WR: per-kernel workspace limit")
    ap.add_argument("--mode", default="wr", choices=["wr", "wd"])
    ap.add_argument("--total-mib", type=int, default=2544, help="WD: network-wide workspace budget")
    ap.add_argument("--ref-sample", type=int, default=0, help="samples per step (0: one per host core, <= 64)")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a replayed CUDA graph")
    ap.add_argument("--db", default=None, help="cost-table CSV to reuse / extend")
    ap.add_argument("--dist-eager", action="store_true",
                    help="N > 1: eager launches with per-layer all-reduces overlapping the backward pass "
                         "(default: graph replay + one bucketed all-reduce per step)")
    ap.add_argument("--plan-only", action="store_true",
                    help="benchmark and plan (writing --db), print the plans as one JSON line, exit")
    ap.add_argument("--bf-stream", type=int, default=2,
                    help="k >= 1: each BackwardFilter on one of k side streams (BF_i on stream i % k), "
                         "overlapping the BackwardData chain (both arms); 0: one stream")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    quiet_stdout()
    cores = os.cpu_count() or 1
    args.ref_sample = args.ref_sample or min(64, cores)
    args.cpu_sample = args.cpu_sample or min(64, cores)
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    from paper_1804_04806_b200 import Handle, OP_NAMES
    from paper_1804_04806_b200._lib import lib
    from paper_1804_04806_b200.network import ConvStack

    rank, world, local = env_rank()
    # under torchrun (WORLD_SIZE set) the NCCL data-parallel step runs at
    # every world size, 1 included: the same path the N > 1 runs take
    dist_on = "WORLD_SIZE" in os.environ
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if dist_on:
        torch.distributed.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    net_path = os.path.join(ROOT, "configs", args.net + ".net")
    limit = args.limit_mib * MiB
    stack = ConvStack(net_path, 256, dev)
    # one cost-table file per rank: rank 0 benchmarks into `db`, the others
    # receive its rows through share_cost_table into their own copy (a shared
    # path would let a non-zero rank truncate rank 0's table mid-flush)
    db = args.db or os.path.join(tempfile.gettempdir(), f"ucudnn_bench_{os.getpid()}.csv")
    if rank != 0:
        db = f"{db}.rank{rank}"

    # plan: benchmark every (algorithm x micro-batch) on the device, WR DP
    t0 = time.perf_counter()
    if dist_on:
        # rank 0 benchmarks; every rank plans from its table -> identical plans
        from paper_1804_04806_b200.network import share_cost_table
        if rank == 0:
            h0 = Handle(policy=args.policy, mode="wr", database=db, stream=stream.cuda_stream)
            stack.plan(h0, limit)
            h0.flush_database()
            h0.close()
        torch.distributed.barrier()
        share_cost_table(db)
    if args.mode == "wd":
        # WD: Get*Algorithm registers every kernel, one ILP divides
        # the budget, the library owns the arena; the undivided baseline gets
        # budget / #kernels each (harness.hpp:71-80)
        total = args.total_mib * MiB
        h = Handle(policy=args.policy, mode="wd", total_workspace=total, database=db, stream=stream.cuda_stream)
        stack.plan(h, 0)
        h.optimize_network()
        limit = total // len(stack.kernels())
    else:
        h = Handle(policy=args.policy, mode="wr", database=db, stream=stream.cuda_stream)
        stack.plan(h, limit)
    h.flush_database()
    plan_s = time.perf_counter() - t0
    plans = {f"{stack.layers[i].name}/{OP_NAMES[op]}": h.plan(a) for (i, op), a in stack.algos.items()}
    if args.plan_only:
        if rank == 0:
            emit({"net": args.net, "mode": args.mode, "policy": args.policy, "db": db,
                  "plan_seconds": round(plan_s, 1),
                  "plans": {k: "+".join(f"{a}@{b}" for a, b in v) for k, v in plans.items()}})
        return
    base = Handle(policy="undivided", mode="wr", database=db, stream=stream.cuda_stream)
    base_stack_algos = {}
    for (i, op) in stack.kernels():
        base_stack_algos[(i, op)] = base.get_algorithm(op, stack.layers[i].shape, limit)
    base_plans = {f"{stack.layers[i].name}/{OP_NAMES[op]}": base.plan(a) for (i, op), a in base_stack_algos.items()}
    # the caller's WR workspace must cover the undivided plans too (in WD mode
    # the planned handle itself needs none: it owns its arena)
    need = max(base.workspace_size(a, op, stack.layers[i].shape) for (i, op), a in base_stack_algos.items())
    if need // 4 + 64 > stack.ws.numel():
        stack.ws = torch.empty(need // 4 + 64, dtype=torch.float32, device=dev)
        stack.ws_bf = torch.empty(need // 4 + 64, dtype=torch.float32, device=dev)
        stack.ws_bf_extra = []

    # Data parallel with graphs (the default): every layer's dW lives in one
    # flat buffer, the 15 planned calls of a step are one CUDA graph, and one
    # bucketed NCCL all-reduce of all the dW (9.9 MB for AlexNet) follows each
    # replay on the compute stream. --dist-eager instead issues the planned
    # calls eagerly with a per-layer all-reduce on a side stream right after
    # each layer's last BackwardFilter micro-batch (ConvStack.step(comm=...)).
    graph_dist = dist_on and not args.no_graph and not args.dist_eager
    flat_dw = None
    if graph_dist:
        sizes = [t["dw"].numel() for t in stack.t]
        flat_dw = torch.empty(sum(sizes), dtype=torch.float32, device=dev)
        off = 0
        for t, n_ in zip(stack.t, sizes):
            t["dw"] = flat_dw[off:off + n_].view_as(t["dw"])
            off += n_
    comm = torch.distributed.group.WORLD if dist_on and not graph_dist else None
    comm_stream = torch.cuda.Stream(dev) if comm is not None else None

    bf_stream = [torch.cuda.Stream(dev) for _ in range(args.bf_stream)] if args.bf_stream else None

    def step_ours():
        stack.step(h, comm, comm_stream, bf_stream=bf_stream)

    ours_algos = stack.algos

    def step_base():
        stack.algos = base_stack_algos
        stack.step(base, comm, comm_stream, bf_stream=bf_stream)
        stack.algos = ours_algos

    # Capture the 15 planned C-ABI calls once into a CUDA graph and replay it,
    # which removes the host launch gaps between the ~140 small kernels; under
    # data parallelism the bucketed all-reduce follows each replay.
    def as_graph(fn, handle):
        if (dist_on and not graph_dist) or args.no_graph:
            n0 = lib().ucudnnGetLaunchCount()
            fn()
            torch.cuda.synchronize(dev)
            return fn, lib().ucudnnGetLaunchCount() - n0
        cs = torch.cuda.Stream(dev)
        handle.set_stream(cs.cuda_stream)
        with torch.cuda.stream(cs):
            fn()  # warm (first-call attribute setting, filter packing)
        cs.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = lib().ucudnnGetLaunchCount()
        with torch.cuda.graph(g, stream=cs):
            fn()
        per_step = lib().ucudnnGetLaunchCount() - n0
        handle.set_stream(stream.cuda_stream)
        if graph_dist:
            def replay_and_reduce():
                g.replay()
                torch.distributed.all_reduce(flat_dw, op=torch.distributed.ReduceOp.SUM)
            return replay_and_reduce, per_step
        return g.replay, per_step

    run_ours, launches_per_step = as_graph(step_ours, h)
    run_base, _ = as_graph(step_base, base)
    sampler = ClockSampler(local) if rank == 0 else None
    ms = timed(run_ours, args.steps, args.warmup, dev, dist_on)
    clocks = sampler.stop() if sampler else None
    ms_base = timed(run_base, args.steps, args.warmup, dev, dist_on)

    # per-kernel device times of our plan (dominant kernel -> roofline)
    evs = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in stack.kernels()}
    per = {k: [] for k in stack.kernels()}
    for it in range(3 + 5):
        stack.step(h, events=evs)
        torch.cuda.synchronize(dev)
        if it >= 3:
            for k, (a, b) in evs.items():
                per[k].append(a.elapsed_time(b))
    per_ms = {k: statistics.median(v) for k, v in per.items()}
    dom = max(per_ms, key=per_ms.get)
    dom_flops = stack.layers[dom[0]].shape.flops()
    dom_tflops = dom_flops / (per_ms[dom] * 1e-3) / 1e12
    peak = tf32_peak(dev) if rank == 0 else None
    traffic = dom_traffic(f"{stack.layers[dom[0]].name}/{OP_NAMES[dom[1]]}",
                          "+".join(f"{a}@{b}" for a, b in h.plan(stack.algos[dom])))

    # end-to-end through the public API with host buffers: H2D of the step's
    # inputs (conv1 input images + top-layer output gradient), 15 planned
    # convolutions, D2H of every filter gradient
    x_host = stack.t[0]["x"].cpu().pin_memory()
    dy_host = stack.t[-1]["dy"].cpu().pin_memory()
    dw_host = [t["dw"].cpu().pin_memory() for t in stack.t]
    h2d = x_host.numel() * 4 + dy_host.numel() * 4
    d2h = sum(d.numel() * 4 for d in dw_host)

    # Input pipeline as a training loop runs it: the next step's inputs (conv1
    # images + top-layer output gradient) are copied host -> device on an H2D
    # stream into the other half of a double buffer while this step computes
    # (a data loader's pinned-memory prefetch); each dW goes device -> host on
    # a D2H stream right after its BackwardFilter. Every step issues exactly
    # one H2D of its successor's inputs and one D2H of its dWs, so the timed
    # region of K steps carries K H2Ds and K D2Hs; the step ends when its D2Hs
    # are done. PCIe is full duplex, hence separate H2D / D2H streams.
    h2d_stream, d2h_stream = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    xbuf = [stack.t[0]["x"], torch.empty_like(stack.t[0]["x"])]
    dybuf = [stack.t[-1]["dy"], torch.empty_like(stack.t[-1]["dy"])]
    state = {"k": 0, "ready": None, "done": None}

    def prefetch(k):
        # inputs of step k into buffer k % 2, once step k - 2 (its last user) is done
        if state["done"] is not None:
            h2d_stream.wait_event(state["done"])
        with torch.cuda.stream(h2d_stream):
            xbuf[k % 2].copy_(x_host, non_blocking=True)
            dybuf[k % 2].copy_(dy_host, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(h2d_stream)
        return ev

    def step_e2e():
        cur = torch.cuda.current_stream(dev)
        k = state["k"]
        if state["ready"] is None:
            state["ready"] = prefetch(k)
        ready = state["ready"]
        stack.t[0]["x"], stack.t[-1]["dy"] = xbuf[k % 2], dybuf[k % 2]
        cur.wait_event(ready)
        nxt = prefetch(k + 1)

        def on_dw(i, st):
            ev = torch.cuda.Event()
            ev.record(st)
            d2h_stream.wait_event(ev)
            with torch.cuda.stream(d2h_stream):
                dw_host[i].copy_(stack.t[i]["dw"], non_blocking=True)

        stack.step(h, comm, comm_stream, on_dw=None if dist_on else on_dw, bf_stream=bf_stream)
        if dist_on:
            if graph_dist:
                torch.distributed.all_reduce(flat_dw, op=torch.distributed.ReduceOp.SUM)
            for d, t in zip(dw_host, stack.t):
                d.copy_(t["dw"], non_blocking=True)
        cur.wait_stream(d2h_stream)
        done = torch.cuda.Event()
        done.record(cur)
        state.update(k=k + 1, ready=nxt, done=done)

    def e2e_body(k):
        # graph body of step k: fork the H2D of step k+1's inputs into buffer
        # (k+1) % 2, compute on buffer k % 2 with each dW's D2H forked after
        # its BackwardFilter, join everything. Consecutive replays on one
        # stream serialise whole graphs, so step k+1 starts after step k's
        # prefetch landed and step k's last use of the buffer it overwrites.
        cur = torch.cuda.current_stream(dev)
        h2d_stream.wait_stream(cur)
        with torch.cuda.stream(h2d_stream):
            xbuf[(k + 1) % 2].copy_(x_host, non_blocking=True)
            dybuf[(k + 1) % 2].copy_(dy_host, non_blocking=True)
        stack.t[0]["x"], stack.t[-1]["dy"] = xbuf[k % 2], dybuf[k % 2]

        def on_dw(i, st):
            d2h_stream.wait_stream(st)
            with torch.cuda.stream(d2h_stream):
                dw_host[i].copy_(stack.t[i]["dw"], non_blocking=True)

        stack.step(h, on_dw=on_dw, bf_stream=bf_stream)
        cur.wait_stream(d2h_stream)
        cur.wait_stream(h2d_stream)

    if dist_on or args.no_graph:
        ms_e2e = timed(step_e2e, args.steps, args.warmup, dev, dist_on)
        e2e_launch = "eager C-ABI launches"
    else:
        # N = 1: the same pipeline replayed as two CUDA graphs (one per
        # buffer parity), like the device-timed arm
        cs = torch.cuda.Stream(dev)
        h.set_stream(cs.cuda_stream)
        with torch.cuda.stream(cs):
            xbuf[0].copy_(x_host, non_blocking=True)
            dybuf[0].copy_(dy_host, non_blocking=True)
            e2e_body(0)  # warm
        cs.synchronize()
        graphs = []
        for k in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                e2e_body(k)
            graphs.append(g)
        h.set_stream(stream.cuda_stream)
        with torch.cuda.stream(cs):
            xbuf[0].copy_(x_host, non_blocking=True)
            dybuf[0].copy_(dy_host, non_blocking=True)
        cs.synchronize()
        rep = {"k": 0}

        def replay_e2e():
            graphs[rep["k"] % 2].replay()
            rep["k"] += 1

        # more warm-up than the device arm: the first replays pay pinned-host
        # first-touch / PCIe ramp costs (e2e spread 3.75-4.36 ms at W = 5)
        ms_e2e = timed(replay_e2e, args.steps, max(args.warmup, 12), dev, dist_on)
        e2e_launch = "two CUDA graphs (one per input-buffer parity) replayed alternately"
    torch.cuda.synchronize(dev)
    stack.t[0]["x"], stack.t[-1]["dy"] = xbuf[0], dybuf[0]

    if rank == 0:
        cpu = None
        if not args.no_cpu:
            sec, cpu_ms, kind = cpu_reference(net_path, args.cpu_sample, os.cpu_count() or 1)
            cpu = {"value": round(cpu_ms, 1), "unit": "ms/iter", "cores": os.cpu_count(), "kind": kind,
                   "cpu_model": cpu_model(),
                   "sample": f"{args.cpu_sample} of 256 samples of each of the 15 kernels ({sec:.1f} s), "
                             f"x{256 // args.cpu_sample}"}
        total_flops = stack.flops()
        line = {
            "metric": METRIC if (args.net == "alexnet" and args.mode == "wr" and args.limit_mib == 64) else
            f"{args.net} bs256 conv fwd+bwd ms/iter ({args.mode.upper()}, "
            f"{args.limit_mib if args.mode == 'wr' else args.total_mib} MiB); speedup vs undivided",
            "value": round(ms, 4), "unit": "ms/iter", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "tf32", "data": "synthetic (N(0,1) activations, He-init filters)",
            "speedup_vs_undivided": round(ms_base / ms, 4), "undivided_ms_per_step": round(ms_base, 4),
            "images_per_s": round(256 * world / (ms * 1e-3), 1),
            "tflops_effective": round(total_flops / (ms * 1e-3) / 1e12, 2),
            "config": {"workload": f"{args.net} conv layers, Forward + BackwardData + BackwardFilter "
                                   f"({len(stack.kernels())} kernels), batch 256 per GPU", "net": args.net,
                       "global_batch": 256 * world,
                       "ws_limit_bytes": limit, "mode": args.mode, "policy": args.policy,
                       "total_workspace_bytes": args.total_mib * MiB if args.mode == "wd" else None,
                       "parallelism": f"dp{world}", "l2": "working set > L2 (no flush needed)",
                       "launch": ("eager" if ((dist_on and not graph_dist) or args.no_graph)
                                  else "cuda-graph replay of the 15 C-ABI calls"
                                  + ("; one bucketed NCCL all-reduce of all dW after each replay" if graph_dist
                                     else ""))
                       + (f"; BackwardFilter on {args.bf_stream} side stream(s) (BF_i on stream i % "
                          f"{args.bf_stream}, after BD_i+1) overlapping the BackwardData chain"
                          if args.bf_stream else "; one stream"),
                       "live_workspaces": (f"{1 + args.bf_stream} caller workspaces of "
                                           f"{stack.ws.numel() * 4 >> 20} MiB each (main stream + one per "
                                           "BackwardFilter side stream); each call stays within the per-kernel "
                                           "limit" if args.mode == "wr" else "library-owned WD arena"),
                       "comm_size": torch.distributed.get_world_size() if dist_on else 1},
            "roofline": {"bound": "tensor", "kernel": f"{stack.layers[dom[0]].name}/{OP_NAMES[dom[1]]}",
                         "achieved": round(dom_tflops, 1), "peak": round(peak, 1), "unit": "TFLOP/s",
                         "frac": round(dom_tflops / peak, 3), "traffic": traffic,
                         "traffic_source": "bytes per call: ncu dram__bytes_read.sum + dram__bytes_write.sum over "
                                           "the call's launches, profiles/r01_traffic.json (same plan)",
                         "peak_source": "cuBLAS TF32 8192^3 GEMM measured in this run"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(ms_e2e, 4), "unit": "ms/iter", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "pipeline": "next step's inputs H2D-prefetched into a double buffer during this step; "
                                "dW D2H after each BackwardFilter; " + e2e_launch},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "plan_seconds": round(plan_s, 1),
            "per_kernel_ms": {f"{stack.layers[i].name}/{OP_NAMES[op]}": round(v, 4) for (i, op), v in per_ms.items()},
            "plans": {k: "+".join(f"{a}@{b}" for a, b in v) for k, v in plans.items()},
            "undivided_plans": {k: "+".join(f"{a}@{b}" for a, b in v) for k, v in base_plans.items()},
        }
        emit(line)
    if dist_on:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
