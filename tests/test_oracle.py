"""The oracle itself: the plain-C fp64 restatement (oracle/conv_oracle.c)
pinned against the reference's execute_plan (golden vectors in
tests/golden/conv_golden.npz, and live against oracle/_ref/ref_conv.so when
it is built), plus the reference's own conv known-answer tests
(test_reference_conv.cpp)."""
import os

import numpy as np
import pytest

from paper_1804_04806_b200 import ConvShape
from tests.oracle_py import conv_ref, inputs_for, rand_int, ref_available

HERE = os.path.dirname(os.path.abspath(__file__))


def test_golden_vectors_from_reference():
    g = np.load(os.path.join(HERE, "golden", "conv_golden.npz"))
    n = 0
    for i in range(3):
        s = ConvShape(*[int(v) for v in g[f"c{i}_shape"]])
        plan = [int(v) for v in g[f"c{i}_plan"]]
        for op in range(3):
            got = conv_ref(op, s, g[f"c{i}_op{op}_a"], g[f"c{i}_op{op}_b"], plan)
            assert np.array_equal(got, g[f"c{i}_op{op}_out"]), (i, op)
            n += 1
    assert n == 9


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref/ref_conv.so not built")
@pytest.mark.parametrize("seed", range(12))
def test_restatement_equals_reference_live(seed):
    rng = np.random.default_rng(seed)
    pick = lambda lo, hi: int(rng.integers(lo, hi + 1))
    R, S = pick(1, 5), pick(1, 5)
    s = ConvShape(pick(1, 4), pick(1, 4), pick(R, 10), pick(S, 10), pick(1, 4), R, S, pick(0, 2), pick(0, 2),
                  pick(1, 3), pick(1, 3))
    plan, left = [], s.N
    while left:
        b = pick(1, left)
        plan.append(b)
        left -= b
    for op in range(3):
        a, b = inputs_for(op, s, rng, integer=True)
        assert np.array_equal(conv_ref(op, s, a, b, plan), conv_ref(op, s, a, b, plan, use_reference=True))


def test_one_by_one_conv_scales():  # test_reference_conv.cpp:73-85
    s = ConvShape(1, 1, 3, 3, 1, 1, 1)
    x = np.arange(9, dtype=np.float64).reshape(1, 1, 3, 3)
    y = conv_ref(0, s, x, np.full((1, 1, 1, 1), 2.0))
    assert np.array_equal(y, 2 * x)


def test_ones_filter_sums_window():  # test_reference_conv.cpp:87-95
    s = ConvShape(1, 1, 3, 3, 1, 3, 3)
    y = conv_ref(0, s, np.ones((1, 1, 3, 3)), np.ones((1, 1, 3, 3)))
    assert y.shape == (1, 1, 1, 1) and y[0, 0, 0, 0] == 9


@pytest.mark.parametrize("stride", [1, 2])
def test_backward_data_is_exact_adjoint(stride):  # test_reference_conv.cpp:116-140
    rng = np.random.default_rng(5)
    s = ConvShape(2, 3, 8, 7, 4, 3, 3, 1, 1, stride, stride)
    x, w, dy = rand_int(rng, (2, 3, 8, 7)), rand_int(rng, (4, 3, 3, 3)), rand_int(rng, (2, 4, s.OH, s.OW))
    lhs = np.sum(conv_ref(0, s, x, w) * dy)
    rhs = np.sum(x * conv_ref(1, s, dy, w))
    assert lhs == rhs


def test_backward_filter_additive_over_samples():  # test_reference_conv.cpp:151-170
    rng = np.random.default_rng(6)
    s = ConvShape(4, 2, 6, 6, 3, 3, 3, 1, 1, 1, 1)
    x, dy = rand_int(rng, (4, 2, 6, 6)), rand_int(rng, (4, 3, 6, 6))
    full = conv_ref(2, s, x, dy)
    parts = conv_ref(2, s.with_batch(1), x[:1], dy[:1]) + conv_ref(2, s.with_batch(3), x[1:], dy[1:])
    assert np.array_equal(full, parts)


def test_backward_filter_finite_differences():  # test_reference_conv.cpp:172-199
    rng = np.random.default_rng(8)
    s = ConvShape(2, 2, 5, 5, 2, 3, 3, 1, 1, 2, 2)
    x, w, dy = rng.standard_normal((2, 2, 5, 5)), rng.standard_normal((2, 2, 3, 3)), \
        rng.standard_normal((2, 2, s.OH, s.OW))
    dw = conv_ref(2, s, x, dy)
    eps = 1e-4
    for idx in [(0, 0, 0, 0), (1, 1, 2, 1), (0, 1, 1, 2)]:
        wp, wm = w.copy(), w.copy()
        wp[idx] += eps
        wm[idx] -= eps
        fd = (np.sum(conv_ref(0, s, x, wp) * dy) - np.sum(conv_ref(0, s, x, wm) * dy)) / (2 * eps)
        assert abs(fd - dw[idx]) <= 1e-5 * max(1.0, abs(dw[idx]))


@pytest.mark.parametrize("op", [0, 1, 2])
def test_every_partition_equals_undivided(op):  # test_reference_conv.cpp:201-262
    rng = np.random.default_rng(10 + op)
    s = ConvShape(5, 2, 6, 5, 3, 3, 3, 1, 0, 2, 1)
    a, b = inputs_for(op, s, rng, integer=True)
    ref = conv_ref(op, s, a, b)
    for plan in ([5], [4, 1], [3, 2], [3, 1, 1], [2, 2, 1], [2, 1, 1, 1], [1] * 5):
        assert np.array_equal(conv_ref(op, s, a, b, plan), ref)
