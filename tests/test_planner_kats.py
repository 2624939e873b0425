"""Known-answer tests restated from the reference's own unit tests.

Each case cites the reference test it restates; expected values are the
reference's. Single-kernel problems go through ucudnnPlanKernels with a cost
table built from the same analytic model the reference test uses
(cost_model.hpp:33-64 on a unit kernel, whose shape factors are 1).
"""
import math
from fractions import Fraction

import pytest

from paper_1804_04806_b200 import (ConvShape, UcudnnError, canonical_cost_table, canonical_time, kernel_hash,
                                   plan_kernels)

HEADER = "kernel_hash,op_type,algorithm,micro_batch,time_us,workspace_bytes,feasible"


# ------------------------------------------------------------ exact times
@pytest.mark.parametrize("text,want", [("27.6", "27.6"), ("0.00000005", "0.00000005"), ("-4.25", "-4.25"),
                                       ("3/4", "0.75"), ("42", "42"), ("1/3", "1/3"), ("6/16", "0.375"),
                                       ("138/5", "27.6"), ("2/4", "0.5")])
def test_time_parse_render(text, want):  # test_rational.cpp:23-48
    assert canonical_time(text) == want


@pytest.mark.parametrize("bad", ["", "1.2.3", "abc", "1/0"])
def test_time_parse_errors(bad):  # test_rational.cpp:29-32
    with pytest.raises(UcudnnError):
        canonical_time(bad)


def test_time_round_trip_random():  # test_rational.cpp:41-46 (own seeds)
    import random
    rnd = random.Random(11)
    for _ in range(300):
        f = Fraction(rnd.randrange(-1000000, 1000000), rnd.randrange(1, 1000))
        s = canonical_time(f"{f.numerator}/{f.denominator}")
        assert Fraction(s) == f if "/" not in s else Fraction(*map(int, s.split("/"))) == f


# ------------------------------------------------------------ cost table
def test_csv_golden_row():  # test_cost_database.cpp:142-148
    row = "00000000000000ab,Forward,2,32,51.475,86769664,1"
    assert canonical_cost_table(HEADER + "\n" + row + "\n") == HEADER + "\n" + row + "\n"


def test_csv_infeasible_rows_are_zeroed_and_sorted():  # cost_database.hpp:216-218, 119-137
    text = HEADER + "\n00000000000000ff,Forward,1,2,9,9,0\n00000000000000ab,BackwardData,0,1,1.50,3,1\n"
    assert canonical_cost_table(text) == (HEADER + "\n00000000000000ab,BackwardData,0,1,1.5,3,1\n"
                                          "00000000000000ff,Forward,1,2,0,0,0\n")


def test_csv_parse_error_names_line():  # test_cost_database.cpp:123-140
    with pytest.raises(UcudnnError, match=":3:"):
        canonical_cost_table(HEADER + "\n00000000000000ab,Forward,2,32,1,1,1\nbroken\n")


# ------------------------------------------------------------ hashes
def test_alexnet_canonical_hashes():  # SURVEY.md Appendix B.1 (reference domain.hpp:159-180)
    want = {"conv1": ("7c6211260c1cd2a9", "edc538d85f9523dc", "40cf41fbca94f6af"),
            "conv2": ("44d072ea5676d5ea", "7fb6ef2a28bb4a5f", "d151e80f0d7b596c"),
            "conv3": ("8e0a3444dd0ac7e5", "327c353807860164", "cd8c963abecc4267"),
            "conv4": ("bb020dd0798caa2a", "9e5e9c0dcfff211f", "f15e989ae08066ac"),
            "conv5": ("9a2c94893e994aaa", "7d8922c6950bc19f", "123411e21b73c62c")}
    shapes = {"conv1": ConvShape(256, 3, 224, 224, 64, 11, 11, 2, 2, 4, 4),
              "conv2": ConvShape(256, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1),
              "conv3": ConvShape(256, 192, 13, 13, 384, 3, 3, 1, 1, 1, 1),
              "conv4": ConvShape(256, 384, 13, 13, 256, 3, 3, 1, 1, 1, 1),
              "conv5": ConvShape(256, 256, 13, 13, 256, 3, 3, 1, 1, 1, 1)}
    for name, s in shapes.items():
        for op in range(3):
            assert f"{kernel_hash(op, s):016x}" == want[name][op]


# ------------------------------------------------------------ planners
def unit_kernel(batch, op=0):
    return [op, batch, 1, 1, 1, 1, 1, 1, 0, 0, 1, 1]


def model_table(kernels, costs, sizes):
    """Cost rows of the analytic model on unit kernels (cost_model.hpp:134-157):
    time = setup + tps * ceil(b/q)*q ; ws = ws_fixed + wsps * b ; b < min -> infeasible."""
    rows = []
    for k in kernels:
        h = kernel_hash(k[0], ConvShape(*k[1:]))
        for alg, (tps, setup, wsps, wsf, minb, q) in enumerate(costs):
            for b in sizes:
                if b < minb:
                    rows.append((h, k[0], alg, b, "0", 0, 0))
                    continue
                t = Fraction(setup) + Fraction(tps) * (math.ceil(b / q) * q)
                rows.append((h, k[0], alg, b, canonical_time(f"{t.numerator}/{t.denominator}"), wsf + wsps * b, 1))
    ops = ["Forward", "BackwardData", "BackwardFilter"]
    return HEADER + "\n" + "".join(f"{h:016x},{ops[o]},{a},{b},{t},{w},{f}\n" for h, o, a, b, t, w, f in rows)


def plan_of(report, kernel=0):
    out = []
    for line in report.splitlines():
        p = line.split()
        if p[:2] == ["kernel", str(kernel)] and p[2] == "micro":
            out.append((int(p[5]), int(p[7])))
    total = next(l.split()[-1] for l in report.splitlines() if l.startswith(f"kernel {kernel} time-us"))
    return out, total


CHEAP_FAST = [("1", "0", 0, 0, 1, 1), ("0.5", "0", 10, 0, 1, 1)]


def test_wr_split_unlocks_fast_algorithm():  # test_wr_optimizer.cpp:38-47
    k = unit_kernel(64)
    rep = plan_kernels("t", [k], ["unit"], model_table([k], CHEAP_FAST, range(1, 65)), "wr", "all", 320)
    assert plan_of(rep) == ([(1, 32), (1, 32)], "32")


def test_wr_time_tie_prefers_fewer_micro_batches():  # test_wr_optimizer.cpp:49-57
    k = unit_kernel(64)
    rep = plan_kernels("t", [k], ["unit"], model_table([k], CHEAP_FAST, range(1, 65)), "wr", "all", 10000)
    assert plan_of(rep) == ([(1, 64)], "32")


def test_wr_undivided_policy():  # test_wr_optimizer.cpp:59-66
    k = unit_kernel(64)
    rep = plan_kernels("t", [k], ["unit"], model_table([k], CHEAP_FAST, [64]), "wr", "undivided", 320)
    assert plan_of(rep) == ([(0, 64)], "64")


def test_wr_quantized_size_repeated():  # test_wr_optimizer.cpp:68-94 (the paper's Fig. 4 case)
    costs = [("2", "0", 0, 0, 1, 1)] * 4 + [("1", "0", 5, 0, 1, 60)]
    k = unit_kernel(180)
    rep = plan_kernels("t", [k], ["unit"], model_table([k], costs, range(1, 181)), "wr", "all", 300)
    assert plan_of(rep) == ([(4, 60)] * 3, "180")


def test_wr_infeasible_message():  # test_wr_optimizer.cpp:96-107
    k = unit_kernel(8, op=2)
    tab = model_table([k], [("1", "0", 0, 10, 1, 1)], range(1, 9))
    with pytest.raises(UcudnnError, match="BackwardFilter") as e:
        plan_kernels("t", [k], ["conv9"], tab, "wr", "all", 5)
    assert "5 bytes" in str(e.value) and "conv9" in str(e.value) and e.value.status == 9


def test_wd_twins_share_front_choose_independently():  # test_wd_optimizer.cpp:279-292
    costs = [("3", "0", 0, 0, 1, 1), ("1", "0", 10, 0, 2, 1)]
    k = unit_kernel(2)
    rep = plan_kernels("t", [k, k], ["twin_a", "twin_b"], model_table([k], costs, [1, 2]), "wd", "all", 20)
    assert "unique-kernel-count 1\n" in rep
    assert "total-time-us 8\n" in rep
    assert plan_of(rep, 0)[0] != plan_of(rep, 1)[0]


def test_wd_infeasible_reports_min_workspace():  # test_wd_optimizer.cpp:191-216 (min achievable total)
    costs = [("1", "0", 4, 0, 1, 1)]
    k = unit_kernel(2)
    tab = model_table([k], costs, [1, 2])
    with pytest.raises(UcudnnError) as e:
        plan_kernels("t", [k, k], ["a", "b"], tab, "wd", "all", 7)
    assert e.value.status == 9 and e.value.min_total_workspace == 8


def test_undivided_speedup_is_one():  # test_network_report.cpp:181-196
    k = unit_kernel(8)
    costs = [("2", "0", 0, 0, 1, 1), ("1", "1", 6, 0, 1, 1)]
    rep = plan_kernels("one", [k], ["a"], model_table([k], costs, [8]), "wr", "undivided", 100)
    assert "speedup 1.000000\n" in rep
