"""Parity at the bench's own scale (AlexNet bs256, SURVEY.md section 8 rows
a17-a20), against the fp64 oracle (reference_conv.hpp:70-278).

The small-shape tests in test_algos_gpu.py never leave the first wave of
tiles; the bench runs up to 1,458 output tiles per call, persistent CTAs
looping over many tiles with double-buffered TMEM, two CTAs per SM, CTA pairs
covering several tiles per cluster, split-K BackwardFilter (one tile's
reduction over several CTAs), 8@128 deferred-finalize runs, and the
zero-workspace implicit GEMM's persistent multi-tile loop. This file runs those paths:

* every feasible algorithm id at micro-batches 64, 128 and 256 for each
  AlexNet layer and op (undivided call on the first b images);
* the 15 planned calls of the bench's plan, replayed from the committed
  B200 cost table (tests/golden/csv/b200_alexnet_pow2_64M.csv), through the
  micro-batch executor;
* one ResNet-18 bs256 pass over its distinct layer shapes (plan replayed
  from tests/golden/csv/b200_resnet18_pow2_64M.csv).

Data are integers (x, w in [-3, 3]; dy in [-1, 1] where a BackwardFilter
reduction is long), exact in TF32, and every fp32 partial sum stays below
2^24 (AlexNet conv1 BF: at most 774,400 products of magnitude <= 9), so
results must equal the oracle bit for bit; Winograd F(4x4) and FFT round in
their transforms and keep their normwise bounds. Forward and BackwardData are
compared on a sample subset (images {0, 63, 64, 127, 128, 255} that exist at
the micro-batch); BackwardFilter on the full reduction. Workspaces and
outputs are surrounded by 64 KiB guard regions whose contents must survive
the call (an overrun into a neighbouring allocation would otherwise pass).
The launch-variant trace (ucudnnDebugGetTrace) records which kernel variants
ran; the last test asserts the bench-scale variants were all exercised.
"""
import functools
import os

import numpy as np
import pytest
import torch

from paper_1804_04806_b200 import ConvShape, Handle, algorithm_workspace
from paper_1804_04806_b200.api import set_trace, take_trace
from paper_1804_04806_b200.network import parse_net
from tests.oracle_py import conv_ref, oracle, out_shape

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "csv")
_, ALEX = parse_net(os.path.join(ROOT, "configs", "alexnet.net"), 256)
SUBSET = [0, 63, 64, 127, 128, 255]
SIZES = [64, 128, 256]
INEXACT = {2: 3e-3, 4: 1e-2}
GUARD = 16384  # floats (64 KiB) on each side of every workspace and output
PATTERN = 1234.5
WS_CAP = 24 << 30
TRACE = []


@pytest.fixture(scope="module", autouse=True)
def _threads():
    oracle().oracle_set_threads(os.cpu_count() or 1)
    set_trace(True)
    yield
    set_trace(False)


def _ints(seed, shape, lo=-3, hi=3):
    return np.random.default_rng(seed).integers(lo, hi + 1, size=shape).astype(np.float32)


@functools.lru_cache(maxsize=None)
def layer_data(net, li, shape):
    """x, w, dy of one layer (float32 host arrays, integers)."""
    s = shape
    x = _ints(100 * li + 1, (s.N, s.C, s.H, s.W))
    w = _ints(100 * li + 2, (s.K, s.C, s.R, s.S))
    # |dy| <= 1 keeps long BackwardFilter reductions (ResNet conv1: 3.2 M
    # products) below 2^24
    dy = _ints(100 * li + 3, (s.N, s.K, s.OH, s.OW), -1, 1) if s.N * s.OH * s.OW > 500_000 else \
        _ints(100 * li + 3, (s.N, s.K, s.OH, s.OW))
    return x, w, dy


@functools.lru_cache(maxsize=None)
def dev_data(net, li, shape):
    return tuple(torch.from_numpy(a).cuda() for a in layer_data(net, li, shape))


def subset(b):
    return [i for i in SUBSET if i < b]


@functools.lru_cache(maxsize=None)
def ref_fbd(net, li, shape, op):
    """Forward / BackwardData oracle on the sample subset (all at N = 256)."""
    x, w, dy = layer_data(net, li, shape)
    idx = subset(shape.N)
    s = shape.with_batch(len(idx))
    a = (x if op == 0 else dy)[idx].astype(np.float64)
    return conv_ref(op, s, a, w.astype(np.float64))


@functools.lru_cache(maxsize=None)
def ref_bf_prefix(net, li, shape, b):
    """BackwardFilter oracle over the first b images (prefix sums reuse the
    smaller prefixes, so all sizes cost one pass over the batch)."""
    x, _, dy = layer_data(net, li, shape)
    prev = [p for p in SIZES if p < b and shape.N >= p]
    lo = prev[-1] if prev else 0
    base = ref_bf_prefix(net, li, shape, lo) if lo else 0.0
    s = shape.with_batch(b - lo)
    return base + conv_ref(2, s, x[lo:b].astype(np.float64), dy[lo:b].astype(np.float64))


def guarded(n_floats, fill=None):
    """(buffer, view): view has n_floats elements, GUARD pattern floats on each side."""
    buf = torch.full((n_floats + 2 * GUARD,), PATTERN, device="cuda")
    view = buf[GUARD:GUARD + n_floats]
    if fill is not None:
        view.copy_(fill.reshape(-1))
    return buf, view


def guards_intact(buf, n_floats):
    head, tail = buf[:GUARD], buf[GUARD + n_floats:]
    return bool(torch.all(head == PATTERN)) and bool(torch.all(tail == PATTERN))


def check(op, got, ref, algs):
    inexact = [INEXACT[a] for a in algs if a in INEXACT]
    if inexact:
        assert np.linalg.norm(got - ref) <= max(inexact) * np.linalg.norm(ref)
    else:
        assert np.array_equal(got, ref), f"max abs diff {np.abs(got - ref).max()}"


def run_call(h, op, s, full, data, algo, ws_bytes, alpha=1.0, beta=0.0):
    """One C-ABI call on the first s.N images; returns the host result
    (subset for F / BD) after checking every guard region."""
    tx, tw, tdy = data
    a = [tx, tdy, tx][op][:s.N]
    b = [tw, tw, tdy[:s.N]][op]
    n_out = int(np.prod(out_shape(op, s)))
    obuf, out = guarded(n_out)
    out = out.view(*out_shape(op, s))
    out.fill_(float("nan") if beta == 0.0 else 0.0)
    wsn = max(ws_bytes, 4) // 4
    wbuf, ws = guarded(wsn)
    take_trace()
    h.run(op, s, a, b, out, algo, ws, alpha, beta)
    torch.cuda.synchronize()
    TRACE.extend(take_trace())
    assert guards_intact(wbuf, wsn), "workspace guard overwritten"
    assert guards_intact(obuf, n_out), "output guard overwritten"
    res = out.cpu().double().numpy()
    return res[subset(s.N)] if op != 2 else res


CASES = [(li, op, b, algo) for li in range(5) for op in range(3) for b in SIZES for algo in range(9)]


def _cid(c):
    li, op, b, algo = c
    return f"{ALEX[li].name}-{['F', 'BD', 'BF'][op]}-b{b}-a{algo}"


@pytest.mark.parametrize("case", CASES, ids=_cid)
def test_alexnet_algorithm_at_scale(cuda, case):
    li, op, b, algo = case
    full = ALEX[li].shape
    s = full.with_batch(b)
    ws_bytes, ok = algorithm_workspace(op, s, algo, b)
    if not ok:
        pytest.skip("infeasible")
    if ws_bytes > WS_CAP:
        pytest.skip(f"workspace {ws_bytes >> 20} MiB")
    got = run_call(Handle(), op, s, full, dev_data("alexnet", li, full), algo, ws_bytes)
    ref = ref_bf_prefix("alexnet", li, full, b) if op == 2 else ref_fbd("alexnet", li, full, op)[:len(subset(b))]
    check(op, got, ref, [algo])


def _replay(net_file, csv_name, limit, shapes):
    path = os.path.join(GOLD, csv_name)
    if not os.path.exists(path):
        pytest.skip(f"{csv_name} not committed")
    return path


@pytest.mark.parametrize("li", range(5), ids=[L.name for L in ALEX])
@pytest.mark.parametrize("op", [0, 1, 2], ids=["F", "BD", "BF"])
def test_alexnet_bench_plan_replayed(cuda, tmp_path, li, op):
    """The bench's planned call (WR 64 MiB, powerOfTwo), planned from the
    committed B200 cost table (no benchmarking: every row is present) and run
    through the micro-batch executor; BF with alpha = 2, beta = -1 against
    integer initial contents (user beta on the first micro-batch only)."""
    src = _replay("alexnet.net", "b200_alexnet_pow2_64M.csv", 64 << 20, ALEX)
    db = tmp_path / "t.csv"
    db.write_text(open(src).read())
    h = Handle(policy="powerOfTwo", database=str(db))
    full = ALEX[li].shape
    algo = h.get_algorithm(op, full, 64 << 20)
    plan = h.plan(algo)
    assert sum(b for _, b in plan) == 256
    ws = h.workspace_size(algo, op, full)
    assert ws <= 64 << 20
    data = dev_data("alexnet", li, full)
    if op == 2:
        init = _ints(999, out_shape(2, full))
        tx, tw, tdy = data
        n_out = init.size
        obuf, out = guarded(n_out, torch.from_numpy(init).cuda())
        out = out.view(*out_shape(2, full))
        wbuf, wsv = guarded(max(ws, 4) // 4)
        take_trace()
        h.run(2, full, tx, tdy, out, algo, wsv, alpha=2.0, beta=-1.0)
        torch.cuda.synchronize()
        TRACE.extend(take_trace())
        assert guards_intact(wbuf, max(ws, 4) // 4) and guards_intact(obuf, n_out)
        got = out.cpu().double().numpy()
        ref = 2.0 * ref_bf_prefix("alexnet", li, full, 256) - init.astype(np.float64)
    else:
        got = run_call(h, op, full, full, data, algo, ws)
        ref = ref_fbd("alexnet", li, full, op)
    check(op, got, ref, [a for a, _ in plan])


_, R18 = parse_net(os.path.join(ROOT, "configs", "resnet18.net"), 256)
R18_DISTINCT = []
for _L in R18:
    if _L.shape not in [m.shape for m in R18_DISTINCT]:
        R18_DISTINCT.append(_L)


@pytest.mark.parametrize("li", range(len(R18_DISTINCT)), ids=[L.name for L in R18_DISTINCT])
@pytest.mark.parametrize("op", [0, 1, 2], ids=["F", "BD", "BF"])
def test_resnet18_plan_at_scale(cuda, tmp_path, li, op):
    """ResNet-18 bs256 (config C3), every distinct layer shape: the WR 64 MiB
    powerOfTwo plan replayed from the committed B200 table, through the
    executor, against the oracle."""
    src = _replay("resnet18.net", "b200_resnet18_pow2_64M.csv", 64 << 20, R18)
    db = tmp_path / "t.csv"
    db.write_text(open(src).read())
    h = Handle(policy="powerOfTwo", database=str(db))
    full = R18_DISTINCT[li].shape
    algo = h.get_algorithm(op, full, 64 << 20)
    plan = h.plan(algo)
    ws = h.workspace_size(algo, op, full)
    got = run_call(h, op, full, full, dev_data("resnet18", li, full), algo, ws)
    ref = ref_bf_prefix("resnet18", li, full, 256) if op == 2 else ref_fbd("resnet18", li, full, op)
    check(op, got, ref, [a for a, _ in plan])


def test_zz_bench_scale_variants_exercised(cuda):
    """The code paths the bench's 3.5 ms consists of actually ran above:
    precomp2 with more tiles than clusters (multi-tile CTA-pair loop), the
    1-SM implicit GEMM at two CTAs per SM, the CTA-pair channels-last
    BackwardFilter, split-K over more units than SMs, and deferred-finalize
    runs (kAccumulate / kDeferFinal across an 8@128 + 8@128 plan), the
    zero-workspace implicit GEMM (algorithm 0) on every AlexNet F / BD, and
    the shared-memory patch kernels of conv1."""
    if not TRACE:
        pytest.skip("run with the rest of this module")

    def kv(line):
        return dict(t.split("=", 1) for t in line.split()[1:] if "=" in t)

    p2 = [kv(l) for l in TRACE if l.startswith("precomp2 ")]
    assert any(int(d["m_tiles"]) * int(d["n_tiles"]) > int(d["clusters"]) for d in p2), "no multi-tile precomp2"
    p1 = [kv(l) for l in TRACE if l.startswith("precomp ")]
    assert any(d["cps"] == "2" for d in p1), "no two-CTA-per-SM precomp"
    bfn = [l for l in TRACE if l.startswith("bfn2 ")]
    assert bfn, "no CTA-pair algorithm-8 BackwardFilter"
    allbf = [kv(l) for l in TRACE if l.startswith(("bfn ", "bfn2 ", "bfl ", "bfl2 "))]
    # split-K: one tile's reduction spread over several persistent CTAs whose
    # fp32 partial sums meet in the RED scratch (units are sized to fill the
    # SMs once, so splits > 1 is the multi-CTA reduction case)
    assert any(int(d["splits"]) > 1 for d in allbf), "no split-K BackwardFilter"
    assert any(d.get("defer") == "1" for d in allbf) and any(d.get("acc") == "1" for d in allbf), \
        "no deferred-finalize run"
    z = [kv(l) for l in TRACE if l.startswith("zgemm ")]
    assert any(int(d["m_tiles"]) * int(d["n_tiles"]) > int(d["grid"]) for d in z), "no multi-tile zgemm"
    # TMA filter (Forward) and the gathered phase sub-filter (BackwardData);
    # the gathered-row Forward path (bmode 1) is reached by the small
    # few-channel shapes of test_algos_gpu.py
    assert {d["bmode"] for d in z} >= {"0", "2"}, "zgemm B paths not exercised"
    assert any(l.startswith("fct fwd ") for l in TRACE), "no TMEM-operand Forward (AlexNet conv1, algorithm 0)"
    assert any(l.startswith("fct bwdf ") for l in TRACE), "no TMEM-operand BackwardFilter (AlexNet conv1)"
    assert any(l.startswith("fct bwdd ") for l in TRACE), "no TMEM-operand BackwardData (AlexNet conv1, algorithm 0)"
    # ResNet-18's plan: stride-1 3x3 BackwardFilter through the TMA-operand
    # TMEM kernel, conv1 BackwardFilter with dy by TMA, conv1 BackwardData in
    # column strips
    assert any(l.startswith("fct bwdf1 ") for l in TRACE), "no stride-1 TMEM-operand BackwardFilter (ResNet-18)"
    assert any(l.startswith("fct bwdf ") and "dtma=1" in l for l in TRACE), "no TMA dy in conv1 BF (ResNet-18)"
    assert any(l.startswith("fct bwdd ") and "strips=2" in l for l in TRACE), "no column strips (ResNet-18 conv1 BD)"
