"""The micro-batch executor through the C ABI (virtual algorithm ids).

A cost table injected through ucudnnSetCostDatabase forces a plan that mixes
algorithms and micro-batch sizes; the executor must then reproduce the
reference execute_plan semantics (reference_conv.hpp:205-278): canonical
micro order, disjoint F/BD slices with per-slice alpha/beta, BF accumulating
with the user's beta on the first micro-batch only.
"""
import numpy as np
import pytest
import torch

from paper_1804_04806_b200 import ConvShape, Handle, algorithm_workspace, kernel_hash
from tests.oracle_py import conv_ref, inputs_for, out_shape

pytestmark = pytest.mark.gpu
HEADER = "kernel_hash,op_type,algorithm,micro_batch,time_us,workspace_bytes,feasible"
OPS = ["Forward", "BackwardData", "BackwardFilter"]


def forced_table(s, op, times):
    """times[alg][b] -> us (missing: infeasible); real workspace sizes."""
    h = kernel_hash(op, s)
    rows = []
    for alg in range(9):
        for b in range(1, s.N + 1):
            t = times.get(alg, {}).get(b)
            ws, ok = algorithm_workspace(op, s, alg, b)
            if t is None or not ok:
                rows.append(f"{h:016x},{OPS[op]},{alg},{b},0,0,0")
            else:
                rows.append(f"{h:016x},{OPS[op]},{alg},{b},{t},{ws},1")
    return HEADER + "\n" + "\n".join(rows) + "\n"


BIG = 10 ** 6
TIMES = {3: {1: 100, 2: 10, 3: BIG, 4: BIG, 5: BIG}, 0: {1: 5, 2: BIG, 3: BIG, 4: BIG, 5: BIG}}


@pytest.mark.parametrize("op", [0, 1, 2], ids=["F", "BD", "BF"])
def test_forced_mixed_plan_matches_oracle(cuda, tmp_path, op):
    s = ConvShape(5, 4, 9, 9, 8, 3, 3, 1, 1, 2, 2)
    db = tmp_path / "t.csv"
    db.write_text(forced_table(s, op, TIMES))
    h = Handle(policy="all", database=str(db))
    algo = h.get_algorithm(op, s, 1 << 30)
    assert h.plan(algo) == [(3, 2), (3, 2), (0, 1)]
    rng = np.random.default_rng(31 + op)
    a, b = inputs_for(op, s, rng, integer=True)
    init = np.random.default_rng(1).integers(-3, 4, size=out_shape(op, s)).astype(np.float64)
    ta, tb = torch.from_numpy(a).float().to(cuda), torch.from_numpy(b).float().to(cuda)
    out = torch.from_numpy(init).float().to(cuda)
    ws = torch.empty(h.workspace_size(algo, op, s) // 4 + 1, device=cuda)
    h.run(op, s, ta, tb, out, algo, ws, alpha=1.0, beta=2.0)
    torch.cuda.synchronize()
    want = conv_ref(op, s, a, b, [2, 2, 1]) + 2.0 * init
    assert np.array_equal(out.cpu().double().numpy(), want)


def assert_plan_result(h, algo, got, ref):
    """Bit-exact on integer data unless the timing put a micro-batch on FFT (2)
    or Winograd F(4x4,3x3) (4): those round in their transforms even on
    integers and are held to their stated normwise bound (test_algos_gpu.TOL)."""
    if {alg for alg, _ in h.plan(algo)} & {2, 4}:
        assert np.linalg.norm(got - ref) <= 1e-2 * np.linalg.norm(ref)
    else:
        assert np.array_equal(got, ref)


def test_wd_mode_plans_network_and_uses_arena(cuda):
    s = ConvShape(4, 16, 10, 10, 32, 3, 3, 1, 1, 1, 1)
    h = Handle(policy="powerOfTwo", mode="wd", total_workspace=64 << 20)
    h.set_benchmark_iterations(1, 2)
    algos = [h.get_algorithm(op, s, 0) for op in range(3)]
    h.optimize_network()
    assert all(h.workspace_size(a, op, s) == 0 for op, a in enumerate(algos))
    rng = np.random.default_rng(4)
    x, w, dy = (inputs_for(0, s, rng)[0], inputs_for(0, s, rng)[1], inputs_for(1, s, rng)[0])
    tx, tw, tdy = (torch.from_numpy(v).float().to(cuda) for v in (x, w, dy))
    outs = [torch.empty(out_shape(op, s), device=cuda) for op in range(3)]
    for op, (ia, ib) in enumerate(((tx, tw), (tdy, tw), (tx, tdy))):
        h.run(op, s, ia, ib, outs[op], algos[op])
    torch.cuda.synchronize()
    for op, (ia, ib) in enumerate(((x, w), (dy, w), (x, dy))):
        assert_plan_result(h, algos[op], outs[op].cpu().double().numpy(), conv_ref(op, s, ia, ib))
    rep = h.machine_report()
    assert "mode wd" in rep and "kernel-count 3" in rep and rep.endswith("end\n")


def test_wr_plan_respects_workspace_limit(cuda):
    s = ConvShape(16, 64, 13, 13, 64, 3, 3, 1, 1, 1, 1)
    h = Handle(policy="powerOfTwo")
    h.set_benchmark_iterations(1, 3)
    for limit in (0, 1 << 20, 64 << 20):
        for op in range(3):
            a = h.get_algorithm(op, s, limit)
            assert h.workspace_size(a, op, s) <= limit
            assert sum(b for _, b in h.plan(a)) == s.N


def test_parallel_benchmark_devices(cuda, tmp_path):
    """ucudnnSetBenchmarkDevices: two benchmark slots (host threads with their
    own streams and scratch; both on device 0 here, the only GPU) fill the
    same cost rows as the sequential benchmarker -- same keys, same
    feasibility and workspace columns -- and the plan they feed runs exactly."""
    import csv
    s = ConvShape(8, 16, 12, 12, 32, 3, 3, 1, 1, 1, 1)
    tables = []
    for devs in ([], [0, 0]):
        db = tmp_path / f"t{len(devs)}.csv"
        h = Handle(policy="all", database=str(db))
        h.set_benchmark_devices(devs)
        algos = [h.get_algorithm(op, s, 1 << 26) for op in (0, 1, 2)]
        h.flush_database()
        rows = list(csv.DictReader(open(db)))
        tables.append({(r["kernel_hash"], r["op_type"], r["algorithm"], r["micro_batch"]):
                       (r["feasible"], r["workspace_bytes"]) for r in rows})
        rng = np.random.default_rng(5)
        for op, algo in enumerate(algos):
            a, b = inputs_for(op, s, rng, integer=True)
            out = torch.zeros(out_shape(op, s), device=cuda)
            ws = torch.empty(max(h.workspace_size(algo, op, s), 4) // 4 + 1, device=cuda)
            h.run(op, s, torch.from_numpy(a).float().to(cuda), torch.from_numpy(b).float().to(cuda), out, algo, ws)
            torch.cuda.synchronize()
            assert_plan_result(h, algo, out.cpu().double().numpy(), conv_ref(op, s, a, b))
        h.close()
    assert tables[0] == tables[1] and len(tables[0]) == 3 * 8 * 9


def test_side_stream_backward_filter_matches_serial(cuda, tmp_path):
    """ConvStack.step with `bf_stream` (every BackwardFilter on a side stream
    with its own workspace, overlapping the BackwardData chain)
    gives bit-identical outputs to the one-stream schedule, eagerly and
    replayed from a CUDA graph."""
    from paper_1804_04806_b200.network import ConvStack
    net = tmp_path / "tiny.net"
    net.write_text("network tiny\nminibatch 8\n"
                   "layer c1 channels=3 size=23x23 filters=32 kernel=5x5 pad=2 stride=2\n"
                   "layer c2 channels=32 size=12x12 filters=64 kernel=3x3 pad=1 stride=1\n"
                   "layer c3 channels=64 size=12x12 filters=64 kernel=3x3 pad=1 stride=1\n")
    stack = ConvStack(str(net), 8, cuda)
    # integer data: exact in TF32 and in any fp32 summation order, so the
    # split-K RED epilogues cannot make the two schedules differ
    gen = torch.Generator(device="cpu").manual_seed(11)
    for t in stack.t:
        for k in ("x", "w", "dy"):
            t[k].copy_(torch.randint(-3, 4, t[k].shape, generator=gen).float())
    h = Handle(policy="powerOfTwo", database=str(tmp_path / "db.csv"))
    stack.plan(h, 1 << 24)
    stack.step(h)
    torch.cuda.synchronize()
    ref = [{k: t[k].clone() for k in ("y", "dx", "dw")} for t in stack.t]
    for t in stack.t:
        for k in ("y", "dx", "dw"):
            t[k].fill_(float("nan"))
    side = torch.cuda.Stream(cuda)
    stack.step(h, bf_stream=side)
    torch.cuda.synchronize()
    for r, t in zip(ref, stack.t):
        for k in r:
            assert torch.equal(r[k], t[k]), k
    for t in stack.t:
        t["dw"].fill_(float("nan"))
    stack.step(h, bf_stream=[side, torch.cuda.Stream(cuda)])  # BF_i on stream i % 2
    torch.cuda.synchronize()
    for r, t in zip(ref, stack.t):
        assert torch.equal(r["dw"], t["dw"])
    cs = torch.cuda.Stream(cuda)
    h.set_stream(cs.cuda_stream)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        stack.step(h, bf_stream=side)
    for t in stack.t:
        t["dw"].fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    for r, t in zip(ref, stack.t):
        assert torch.equal(r["dw"], t["dw"])
    h.close()


@pytest.mark.parametrize("case", ["run-then-other", "run-only"])
def test_bf_deferred_finalize_runs(cuda, tmp_path, case):
    """Algorithm 8 keeps its fp32 partial sums across a run of consecutive
    micro-batches of one BackwardFilter call and finalizes once (kAccumulate /
    kDeferFinal): the run must still apply the user's beta exactly once and
    hand over to a different algorithm with beta = 1 (forced plans
    8@2 + 8@2 + 6@1 and 8@2 + 8@2)."""
    n = 5 if case == "run-then-other" else 4
    s = ConvShape(n, 32, 7, 7, 48, 3, 3, 1, 1, 1, 1)
    times = {8: {2: 4, 1: 3}, 6: {1: 2.5}} if n == 5 else {8: {2: 4}}
    db = tmp_path / "t.csv"
    db.write_text(forced_table(s, 2, times))
    h = Handle(policy="all", database=str(db))
    algo = h.get_algorithm(2, s, 1 << 30)
    want_plan = [(8, 2), (8, 2), (6, 1)] if n == 5 else [(8, 2), (8, 2)]
    assert h.plan(algo) == want_plan
    rng = np.random.default_rng(77)
    a, b = inputs_for(2, s, rng, integer=True)
    init = np.random.default_rng(2).integers(-3, 4, size=out_shape(2, s)).astype(np.float64)
    out = torch.from_numpy(init).float().to(cuda)
    ws = torch.empty(h.workspace_size(algo, 2, s) // 4 + 1, device=cuda)
    h.run(2, s, torch.from_numpy(a).float().to(cuda), torch.from_numpy(b).float().to(cuda), out, algo, ws,
          alpha=2.0, beta=-1.0)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().double().numpy(), 2.0 * conv_ref(2, s, a, b) - init)
