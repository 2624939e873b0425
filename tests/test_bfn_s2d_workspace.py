"""Host-side geometry of algorithm 8 (IMPLICIT_PRECOMP_GEMM_NHWC) BackwardFilter
through the space-to-depth copy (bfnhwc.cu make_geo / bfn_workspace), checked
through the C ABI's workspace query (no GPU needed).

Strided layers with few channels or 1x1 filters run as the stride-1
BackwardFilter of x_s2d[n][i][j][(a*Bw + b)*C + c] = x[n][c][i*sh + a - ph][j*sw + b - pw]
with ceil(R/sh) x ceil(S/sw) taps; the workspace is the [k][row] fp32 partial-sum
scratch + the s2d copy + dy's channels-last copy (none when OH*OW % 4 == 0:
dy is read in place).
"""
import pytest

from paper_1804_04806_b200 import ConvShape, algorithm_workspace


def _a256(b):
    return (b + 255) // 256 * 256


def _ru(a, b):
    return (a + b - 1) // b * b


def expected_ws(s: ConvShape, n: int) -> int:
    oh, ow = s.OH, s.OW
    ah, bw = min(s.sh, s.R), min(s.sw, s.S)
    th, tw = -(-s.R // s.sh), -(-s.S // s.sw)
    cc = ah * bw * s.C
    cp, kp = _ru(cc, 32), _ru(s.K, 32)
    m = th * tw * cp
    # tile choice as make_geo: CTA pairs when 512-row pair tiles pad no more
    # than 256-row tiles; otherwise 1 or 2 sub-tiles of 128 rows
    two = _ru(m, 512) <= _ru(m, 256)
    pair_rows = 256 if two else 128
    if m <= pair_rows:
        msub = 1
    elif two:
        msub = 2
    else:
        msub = 2 if _ru(m, 256) <= _ru(m, 128) else 1
    m_tiles = -(-m // (msub * pair_rows))
    rows_pad = m_tiles * msub * pair_rows
    hq, wq = oh + th - 1, ow + tw - 1
    acc = _a256(s.K * rows_pad * 4)
    x = _a256(n * hq * wq * cp * 4)
    dy = 0 if (oh * ow) % 4 == 0 else _a256(n * oh * ow * kp * 4)
    return acc + x + dy


@pytest.mark.parametrize("s,n", [
    (ConvShape(256, 3, 224, 224, 64, 11, 11, 2, 2, 4, 4), 32),   # AlexNet conv1: 48 -> 64 channels, 3x3 taps
    (ConvShape(256, 3, 224, 224, 64, 7, 7, 3, 3, 2, 2), 16),     # ResNet conv1: 12 -> 32 channels, 4x4 taps, dy in place
    (ConvShape(256, 64, 56, 56, 128, 1, 1, 0, 0, 2, 2), 32),     # 1x1 stride-2 shortcut: a subsampling copy
    (ConvShape(4, 3, 31, 31, 16, 11, 11, 2, 2, 4, 4), 4),        # the GPU test's conv1 geometry
])
def test_s2d_workspace_matches_geometry(s, n):
    ws, ok = algorithm_workspace(2, s, 8, n)
    assert ok
    assert ws == expected_ws(s, n)


def test_s2d_not_used_for_wide_strided_3x3():
    # 3x3 stride 2 with 64 channels would pad 9 taps to 16 (2x2 taps of 4 phases):
    # algorithm 8 declines it; stride-1 channel counts must stay multiples of 32
    assert not algorithm_workspace(2, ConvShape(256, 64, 56, 56, 128, 3, 3, 1, 1, 2, 2), 8, 32)[1]
    assert not algorithm_workspace(2, ConvShape(8, 48, 13, 13, 64, 3, 3, 1, 1, 1, 1), 8, 8)[1]
    # BackwardFilter only
    assert not algorithm_workspace(0, ConvShape(256, 3, 224, 224, 64, 11, 11, 2, 2, 4, 4), 8, 32)[1]
