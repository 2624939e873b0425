"""Every concrete algorithm vs the fp64 oracle, through the C ABI (undivided).

Integer data in [-3, 3] is exact in TF32 and every partial sum here stays
below 2^24, so GEMM-class results must equal the oracle bit-for-bit.
Gaussian data checks the stated TF32 tolerance: normwise relative error
<= 3e-3 (TF32 keeps 10 mantissa bits; accumulation is fp32).
"""
import numpy as np
import pytest
import torch

from paper_1804_04806_b200 import ConvShape, Handle, algorithm_workspace
from tests.oracle_py import conv_ref, inputs_for, out_shape

pytestmark = pytest.mark.gpu

SHAPES = [
    ConvShape(2, 3, 11, 11, 16, 3, 3, 1, 1, 1, 1),
    ConvShape(3, 8, 9, 7, 24, 3, 3, 0, 0, 1, 1),
    ConvShape(2, 5, 13, 13, 7, 5, 5, 2, 2, 1, 1),
    ConvShape(2, 3, 31, 31, 16, 11, 11, 2, 2, 4, 4),      # AlexNet conv1 geometry
    ConvShape(2, 16, 14, 14, 32, 1, 1, 0, 0, 2, 2),       # ResNet 1x1 s2 shortcut
    ConvShape(2, 16, 15, 15, 32, 3, 3, 1, 1, 2, 2),       # ResNet 3x3 s2
    ConvShape(1, 3, 30, 30, 64, 7, 7, 3, 3, 2, 2),        # ResNet conv1 geometry
    ConvShape(4, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1),      # AlexNet conv2
    ConvShape(2, 192, 13, 13, 384, 3, 3, 1, 1, 1, 1),     # AlexNet conv3 (N tiles of 192)
    ConvShape(2, 40, 6, 6, 300, 3, 3, 1, 1, 1, 1),        # ragged tiles
    ConvShape(3, 64, 7, 7, 64, 3, 3, 1, 1, 1, 1),         # ResNet l4-like spatial size
    ConvShape(2, 64, 14, 14, 32, 1, 1, 0, 0, 1, 1),       # 1x1 stride 1: BF reads x / dy in place
    ConvShape(3, 32, 7, 7, 160, 1, 1, 0, 0, 1, 1),        # 1x1 stride 1, 49-pixel planes (re-laid)
    ConvShape(2, 3, 36, 36, 16, 11, 11, 2, 2, 4, 4),      # conv1 geometry, W % 4 == 0 (float4 s2d loads)
    ConvShape(2, 3, 32, 32, 64, 7, 7, 3, 3, 2, 2),        # ResNet conv1 geometry, W % 4 == 0
    ConvShape(3, 36, 12, 12, 40, 1, 1, 0, 0, 1, 1),       # 1x1 s1 (TMA plane GEMM): C % 32 != 0, partial plane tile
    ConvShape(2, 64, 56, 56, 256, 1, 1, 0, 0, 1, 1),      # ResNet-50 res2 1x1: 25 plane tiles per image
    ConvShape(2, 64, 56, 56, 128, 1, 1, 0, 0, 2, 2),      # ResNet-50 res3a_1 projection: 1x1 stride 2 (4-D TMA map)
    ConvShape(3, 36, 12, 12, 40, 1, 1, 0, 0, 2, 2),       # 1x1 s2, OW < 32: several output rows per tile
    ConvShape(2, 32, 15, 16, 16, 1, 1, 0, 0, 2, 2),       # 1x1 s2, odd H: last dx row of each 2x2 block missing
    ConvShape(2, 3, 8, 8, 16, 3, 3, 0, 0, 3, 3),          # kernel == stride, trailing column unread (s2d row pitch)
    ConvShape(2, 3, 36, 36, 16, 8, 8, 0, 0, 8, 8),        # kernel == stride, W % 4 == 0 (s2d float4 path bound)
]
ALGOS = [0, 1, 2, 3, 4, 5, 6, 7, 8]
# F(4x4,3x3) carries 1/6 and 1/24 in G: not exact in TF32 even on integer data,
# and its transforms amplify TF32 rounding (measured ~3.3e-3 normwise on
# Gaussian data), so it gets a 1e-2 bound instead of the GEMM-class 3e-3.
# FFT rounds in its transforms: tolerance-checked only, at the GEMM bound.
INEXACT = {2, 4}
TOL = {2: 3e-3, 4: 1e-2}


def _sid(s):
    return f"{s.N}x{s.C}x{s.H}x{s.W}-k{s.K}r{s.R}p{s.ph}s{s.sh}"


def run_algo(h, op, s, a, b, dev, algo, alpha=1.0, beta=0.0, init=None):
    ws_bytes, ok = algorithm_workspace(op, s, algo, s.N)
    if not ok:
        pytest.skip(f"algorithm {algo} does not implement op {op} for {s}")
    ta, tb = torch.from_numpy(a).float().to(dev), torch.from_numpy(b).float().to(dev)
    out = torch.from_numpy(init).float().to(dev) if init is not None else \
        torch.full(out_shape(op, s), float("nan"), device=dev)
    ws = torch.empty(max(ws_bytes, 4) // 4 + 1, device=dev)
    h.run(op, s, ta, tb, out, algo, ws, alpha, beta)
    torch.cuda.synchronize()
    return out.cpu().double().numpy()


@pytest.mark.parametrize("s", SHAPES, ids=_sid)
@pytest.mark.parametrize("op", [0, 1, 2], ids=["F", "BD", "BF"])
@pytest.mark.parametrize("algo", ALGOS)
def test_integer_bit_exact(cuda, algo, op, s):
    rng = np.random.default_rng(1804 + op)
    a, b = inputs_for(op, s, rng, integer=True)
    got = run_algo(Handle(), op, s, a, b, cuda, algo)
    ref = conv_ref(op, s, a, b)
    if algo in INEXACT:
        assert np.linalg.norm(got - ref) <= TOL[algo] * np.linalg.norm(ref)
        return
    assert np.array_equal(got, ref), f"max abs diff {np.abs(got - ref).max()}"


@pytest.mark.parametrize("s", SHAPES[:9], ids=_sid)
@pytest.mark.parametrize("op", [0, 1, 2], ids=["F", "BD", "BF"])
@pytest.mark.parametrize("algo", ALGOS)
def test_gaussian_tf32_tolerance(cuda, algo, op, s):
    rng = np.random.default_rng(7 + op)
    a, b = inputs_for(op, s, rng, integer=False)
    got = run_algo(Handle(), op, s, a, b, cuda, algo)
    ref = conv_ref(op, s, a, b)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= TOL.get(algo, 3e-3), err


AB_SHAPES = [
    ConvShape(3, 6, 10, 10, 20, 3, 3, 1, 1, 1, 1),
    ConvShape(2, 16, 14, 14, 32, 1, 1, 0, 0, 2, 2),   # BD: dx phases without taps get beta * dx
    ConvShape(2, 3, 31, 31, 16, 11, 11, 2, 2, 4, 4),  # stride-phase BD / space-to-depth F
]


@pytest.mark.parametrize("s", AB_SHAPES, ids=_sid)
@pytest.mark.parametrize("op", [0, 1, 2], ids=["F", "BD", "BF"])
@pytest.mark.parametrize("algo", ALGOS)
def test_alpha_beta(cuda, algo, op, s):
    rng = np.random.default_rng(3)
    a, b = inputs_for(op, s, rng, integer=True)
    init = np.random.default_rng(4).integers(-3, 4, size=out_shape(op, s)).astype(np.float64)
    got = run_algo(Handle(), op, s, a, b, cuda, algo, alpha=2.0, beta=-1.0, init=init)
    ref = 2.0 * conv_ref(op, s, a, b) - init
    if algo in INEXACT:
        assert np.linalg.norm(got - ref) <= TOL[algo] * np.linalg.norm(ref)
        return
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("spec", ["2 3 31 31 16 11 11 2 4", "2 3 40 40 64 7 7 3 2", "2 16 14 14 32 1 1 0 2"])
def test_experimental_bd_scatter(cuda, spec):
    """The GEMM + col2im BackwardData kernel (bdscatter.cu) is off by default
    (UCUDNN_TUNE=bds=1 enables it as algorithm 6 for op 1); the knob is read
    once per process, so run it in a child."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, UCUDNN_TUNE="bds=1")
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "one_small.py"), *spec.split(), "1", "6"],
                         env=env, capture_output=True, text=True, timeout=300)
    assert "exact True" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("spec", ["3 64 13 13 96 3 3 1 1 0", "3 64 13 13 96 3 3 1 1 1", "2 96 28 28 64 3 3 1 2 1",
                                  "2 128 28 28 64 1 1 0 2 1", "2 96 27 27 64 5 5 2 1 0"])
def test_precomp_sliced(cuda, spec):
    """IMPLICIT_PRECOMP_GEMM_SLICED (algorithm 7) splits the reduction channels
    once the channels-last copy passes a cap; a 64 KiB cap (read once per
    process, so in a child) forces 2-3 slices on these small shapes."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, UCUDNN_TUNE="slice_cap_kib=64")
    v = spec.split()
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "one_small.py"), *v[:9], v[9], "7"],
                         env=env, capture_output=True, text=True, timeout=300)
    assert "exact True" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("tune", ["", "bfn2=1,bfn_msub=1", "bfn2=1,bfn_msub=2", "bfn2=0,bfn_msub=1", "bfn2=0,bfn_msub=2",
                                  "bfn_px=64", "bfn_dyd=0", "bfn_dyd=0,bfn2=1"])
@pytest.mark.parametrize("spec", ["2 128 9 9 64 2 2 0 1", "3 64 11 13 96 3 3 1 1", "2 96 7 7 200 5 5 2 1",
                                  "1 32 6 6 40 1 1 0 1", "3 64 12 12 64 3 3 1 1", "2 32 20 20 80 3 3 1 1",
                                  # strided layers through the space-to-depth copy
                                  "2 3 31 31 16 11 11 2 4", "2 3 36 36 70 7 7 3 2", "2 64 14 14 32 1 1 0 2"])
def test_bf_nhwc_variants(cuda, spec, tune):
    """IMPLICIT_PRECOMP_GEMM_NHWC (algorithm 8) BackwardFilter: the 1-SM
    kernel with one or two MMA sub-tiles per CTA, the CTA-pair kernel, and
    64-pixel ring stages, dy read in place (OH*OW % 4 == 0) or through its
    channels-last copy, forced through UCUDNN_TUNE (read once per process,
    so each runs in a child); bit-exact against the fp64 oracle on integer
    data (ragged K, N*P or OH*OW not a multiple of 32, rows past R*S*C;
    strided few-channel and 1x1 layers through the space-to-depth copy)."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, UCUDNN_TUNE=tune)
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "one_small.py"), *spec.split(), "2", "8"],
                         env=env, capture_output=True, text=True, timeout=300)
    assert "exact True" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("tune,spec", [("bfl_xmn=1", "2 3 31 31 16 11 11 2 4 2 6"),
                                       ("bfl_xmn=1", "2 3 36 36 70 7 7 3 2 2 6"),
                                       ("bfl_xmn=1", "3 5 13 13 7 5 5 2 1 2 6"),
                                       ("z=0", "2 3 31 31 16 11 11 2 4 0 0"),
                                       ("z=0", "2 16 15 15 32 3 3 1 2 1 0"),
                                       ("z=0", "3 8 9 7 24 3 3 0 1 2 0"),
                                       ("z_msub=2", "3 5 13 13 7 5 5 2 1 0 0"),
                                       ("z_msub=2", "3 5 13 13 7 5 5 2 1 1 0"),
                                       ("z_msub=2", "2 3 31 31 16 11 11 2 4 1 0"),
                                       ("z_msub=2", "4 40 9 9 300 3 3 1 1 0 0"),
                                       ("z_msub=2", "4 40 9 9 300 3 3 1 1 1 0"),
                                       ("z_bres=1", "2 3 31 31 16 11 11 2 4 1 0"),
                                       ("z_bres=1", "2 3 30 30 64 7 7 3 2 1 0"),
                                       ("z_bres=1", "3 5 13 13 7 5 5 2 1 1 0"),
                                       ("fct_bd=0", "2 3 31 31 16 11 11 2 4 1 0"),
                                       ("fct_bd=0", "2 3 36 36 70 7 7 3 2 1 0"),
                                       ("fct_bd_ring=18", "3 3 63 63 20 11 11 1 4 1 0"),
                                       ("fct_bd_ring=15", "2 3 36 36 64 7 7 3 2 1 0"),
                                       ("fct_bd_pair=1", "2 3 31 31 16 11 11 2 4 1 0"),
                                       ("fct_bd_pair=1", "3 3 47 51 64 11 11 2 4 1 0"),
                                       ("fct_bd_pair=1", "2 3 100 140 32 7 7 3 2 1 0"),
                                       ("fct_bd_pair=1", "1 3 45 45 8 11 11 0 4 1 0"),
                                       ("fct_bd_strips=2", "2 3 36 36 64 7 7 3 2 1 0"),
                                       ("fct_bd_strips=3", "3 3 47 51 64 11 11 2 4 1 0"),
                                       ("", "2 3 100 140 32 7 7 3 2 1 0"),
                                       ("", "3 64 12 12 64 3 3 1 1 2 6"),
                                       ("", "2 32 16 16 48 3 3 1 1 2 6"),
                                       ("", "3 96 8 8 64 5 5 2 1 2 6"),
                                       ("", "1 256 8 8 128 3 3 1 1 2 6"),
                                       ("fct_bf1_ring=4", "3 64 12 12 64 3 3 1 1 2 6"),
                                       ("fct_bf1_ring=6", "3 96 8 8 64 5 5 2 1 2 6"),
                                       ("fct_bf1=0", "3 64 12 12 64 3 3 1 1 2 6"),
                                       ("", "2 64 56 56 128 1 1 0 2 0 5"),
                                       ("", "2 64 15 15 32 1 1 0 2 0 5"),
                                       ("pc_subsample=0", "2 64 56 56 128 1 1 0 2 0 5"),
                                       ("fct1=1", "2 64 27 27 192 5 5 2 1 0 7"),
                                       ("fct1=1", "2 64 27 27 192 5 5 2 1 1 7"),
                                       ("fct1=1", "3 64 12 12 64 3 3 1 1 1 7"),
                                       ("fct1=1", "2 64 28 28 128 3 3 1 1 1 7"),
                                       ("fct1=1", "1 64 56 56 64 3 3 1 1 0 0"),
                                       ("fct_bf_dtma=0", "4 3 48 48 64 7 7 3 2 2 6"),
                                       ("", "4 3 48 48 64 7 7 3 2 2 6"),
                                       ("fct_bf=0", "2 3 31 31 16 11 11 2 4 2 6"),
                                       ("fct_bf=0", "2 3 36 36 70 7 7 3 2 2 6"),
                                       ("fct_bf_ring=15", "3 3 63 63 20 11 11 1 4 2 6"),
                                       ("fct_bf_ring=9", "3 3 36 36 64 7 7 3 2 2 6"),
                                       ("fct_epi=8", "2 3 31 31 16 11 11 2 4 0 0"),
                                       ("fct_epi=8", "2 3 36 36 70 7 7 3 2 0 0"),
                                       ("fct_epi=4", "2 3 224 224 64 7 7 3 2 0 0"),
                                       ("fct=0", "2 3 31 31 16 11 11 2 4 0 0"),
                                       ("fct=0", "2 3 36 36 70 7 7 3 2 0 0"),
                                       ("fct_ring=79", "4 3 63 63 20 11 11 1 4 0 0"),
                                       ("fct_ring=33", "3 3 36 36 64 7 7 3 2 0 0"),
                                       ("pc2_msub=2", "3 64 13 13 192 3 3 1 1 0 5"),
                                       ("pc2_msub=2", "5 64 27 27 192 5 5 2 1 0 5"),
                                       ("pc2_msub=2", "3 256 13 13 64 3 3 1 1 1 5"),
                                       ("pc2_msub=2", "2 32 28 28 128 3 3 1 2 0 5"),
                                       ("strip=1", "3 64 12 12 64 3 3 1 1 0 5"),
                                       ("strip=1", "3 64 12 12 64 3 3 1 1 1 5"),
                                       ("strip=1,strip_msub=4", "5 64 27 27 40 5 5 2 1 1 5"),
                                       ("strip=1,strip_msub=4", "3 32 9 9 64 3 3 1 1 0 5"),
                                       ("strip=1,strip_msub=1", "3 40 9 9 70 3 3 1 1 0 5"),
                                       ("strip=1", "2 16 15 15 32 3 3 1 2 1 5"),
                                       ("sswap=1", "3 64 12 12 64 3 3 1 1 1 5"),
                                       ("", "2 64 16 16 128 3 3 1 2 1 5"),
                                       ("", "3 32 9 9 64 3 3 1 2 1 5"),
                                       ("", "3 64 15 17 64 3 3 1 2 1 5"),
                                       ("ph32=0", "2 64 16 16 128 3 3 1 2 1 5"),
                                       ("strip=1", "2 64 16 16 128 3 3 1 2 1 5")])
def test_knob_variants(cuda, tune, spec):
    """Variants the default shapes here do not reach, kept exact: the gather
    BackwardFilter with MN-major x rows (bfl_xmn=1), algorithm 0's
    SIMT-gather fallback (z=0, shapes the tcgen05 kernel does not take) and
    its two-sub-tile mode (z_msub=2, chosen automatically only at large
    batch), resident-filter BackwardData (z_bres=1) and the CTA-pair implicit
    GEMM's two pair sub-tiles per tile (pc2_msub=2, 512 rows, BN=256 with one
    accumulator set), the shared-memory-patch Forward behind the TMEM-operand
    one (fct=0), the shared-memory-patch BackwardFilter behind the TMEM-operand
    one (fct_bf=0), the zero-workspace gather BackwardData behind the
    TMEM-operand one (fct_bd=0), and the TMEM-operand kernels' row rings at
    their minimum depth (fct_ring / fct_bf_ring / fct_bd_ring: loaders wait
    on almost every tile); UCUDNN_TUNE is read
    once per process, so each runs in a child."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, UCUDNN_TUNE=tune)
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "one_small.py"), *spec.split()],
                         env=env, capture_output=True, text=True, timeout=300)
    assert "exact True" in out.stdout, out.stdout + out.stderr
    if tune.startswith("strip=1") or tune == "sswap=1":
        assert "strip swap=" in out.stdout, out.stdout
    if tune == "pc2_msub=2":
        assert "precomp2" in out.stdout and "msub=2" in out.stdout, out.stdout
    if tune.startswith("fct_ring="):
        assert "fct fwd" in out.stdout and tune.replace("fct_", "") in out.stdout, out.stdout
    if tune == "fct_bd_pair=1":
        assert "fct bwdd" in out.stdout and "pair=1" in out.stdout, out.stdout
    if tune.startswith("fct_bd_strips="):
        assert "fct bwdd" in out.stdout and "strips=" + tune.split("=")[1] in out.stdout, out.stdout
    if tune.startswith("fct_bd_ring="):
        assert "fct bwdd" in out.stdout and tune.replace("fct_bd_", "") in out.stdout, out.stdout
    if tune == "" and spec.endswith(" 1 1 0 2 0 5"):
        assert "precomp subsample" in out.stdout, out.stdout
    if spec == "4 3 48 48 64 7 7 3 2 2 6":
        assert ("dtma=0" if tune else "dtma=1") in out.stdout, out.stdout
    if tune == "fct1=1":
        assert "fct1 op=" in out.stdout, out.stdout
    if tune.startswith("fct_bf1_ring=") or (tune == "" and spec.endswith(" 2 6") and int(spec.split()[1]) > 4):
        assert "fct bwdf1" in out.stdout, out.stdout
    if tune.startswith("fct_bf_ring="):
        assert "fct bwdf" in out.stdout and tune.replace("fct_bf_", "") in out.stdout, out.stdout
