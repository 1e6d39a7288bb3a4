"""rhs b = (kron A_d^T) y (Eq. 4's successive mode products,
PAPER.md:68-73, Table 1's up/down-sampling) through the
round-2 kernels against the CPU oracle on seeded inputs:

  * band_mode_product_win_kernel (window-staged, asynchronous copies): chunks
    aligned and not aligned to the outer index, band widths 3..16, windows at
    the matrix edges (zero-filled rows);
  * band_plane2_kernel (the two fastest modes in one plane pass): orders 2-4,
    ragged planes, guards at both edges;
  * the opt-in fused first pass (band_win_last_kernel, TCA_RHS_FUSE1=1) in a
    child process;
  * config 3 at full size (4.0 GB of y) at sampled outputs, and its forward
    model (the expanding chain) at sampled outputs.
Tolerances: fp64 <= 1e-12 relative, fp32 <= 1e-5."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tca():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1001_5460_b200 import tca as t
    return t


def relerr(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300)


# (n, m, basis): oversampling 1.3x-3x (band widths of A_d^T from ~4 to ~13),
# extents that leave ragged window chunks and planes
SHAPES = [
    ((40, 24, 18, 9), (80, 48, 36, 18), "bspline"),       # 2x, order 4
    ((33, 17, 29, 7), (99, 51, 87, 21), "bspline"),       # 3x: wide A^T rows
    ((50, 21, 13), (65, 28, 17), "bspline"),              # 1.3x, order 3
    ((300, 77), (600, 160), "bspline"),                   # order 2 (plane = the whole tensor)
    ((61, 45, 5, 3), (122, 90, 11, 7), "bspline"),        # tiny trailing modes
    ((20, 18, 16), (26, 24, 22), "gauss"),                # dense modes (generic kernels)
]


@pytest.mark.parametrize("n,m,basis", SHAPES)
def test_rhs_and_forward_shapes(n, m, basis, tca):
    A, L = synth.mode_matrices(n, m, basis=basis)
    o = oracle.Operator(A, L, 0.01)
    yd = synth.data(A, n, m, seed=3)
    ref = o.rhs(yd)
    for dt, tdt, tol in (("f64", torch.float64, 1e-12), ("f32", torch.float32, 1e-5)):
        g = tca.Operator(A, L, 0.01, dtype=dt)
        b = g.rhs(torch.from_numpy(yd).to("cuda", tdt))
        torch.cuda.synchronize()
        assert relerr(b.double().cpu().numpy(), ref) <= tol, dt
        # forward model (expanding chain) of a known x, no noise
        x = synth.random_tensor(n, seed=7)
        yf = g.forward_model(torch.from_numpy(x).to("cuda", tdt), sigma=0.0)
        torch.cuda.synchronize()
        assert relerr(yf.double().cpu().numpy(), synth.forward_model(A, x)) <= tol, dt
        g.close()


def test_rhs_fused_first_pass_in_child(tca, tmp_path):
    """TCA_RHS_FUSE1=1 (opt-in): mode 1 and the contiguous last mode in one pass."""
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r})
import oracle, synth
from paper_1001_5460_b200 import tca
worst = 0.0
for n, m in [((40, 24, 18, 9), (80, 48, 36, 18)), ((33, 17, 29, 7), (99, 51, 87, 21)), ((300, 77), (600, 160)),
             ((50, 21, 13), (65, 28, 17))]:
    A, L = synth.mode_matrices(n, m)
    o = oracle.Operator(A, L, 0.01)
    yd = synth.data(A, n, m, seed=3)
    ref = o.rhs(yd)
    for dt, tdt, tol in (("f64", torch.float64, 1e-12), ("f32", torch.float32, 1e-5)):
        g = tca.Operator(A, L, 0.01, dtype=dt)
        b = g.rhs(torch.from_numpy(yd).to("cuda", tdt)).double().cpu().numpy()
        e = np.linalg.norm(b - ref) / np.linalg.norm(ref)
        assert e <= tol, (n, dt, e)
        worst = max(worst, e / tol)
print("ok", worst)
"""
    env = dict(os.environ, TCA_RHS_FUSE1="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok" in r.stdout


def test_rhs_config3_full_size_sampled(tca):
    """Config 3's rhs (y: 256^3 x 30, 4.0 GB fp64) at 64 sampled outputs, each
    computed by the oracle's point evaluation; f64 and f32."""
    c = synth.CONFIGS[3]
    A, L = synth.mode_matrices(c)
    g = tca.Operator(A, L, c.lam)
    y = g.forward_model(None, sigma=synth.NOISE_SIGMA, seed=1)
    b = g.rhs(y)
    rng = np.random.default_rng(11)
    idx = np.stack([rng.integers(0, k, 64) for k in c.n], axis=1)
    idx[:4] = [[0, 0, 0, 0], [c.n[0] - 1, c.n[1] - 1, c.n[2] - 1, c.n[3] - 1], [0, 64, 127, 7], [127, 0, 3, 14]]
    yh = y.cpu().numpy()
    bh = b.cpu().numpy()
    o = oracle.Operator(A, L, c.lam)
    ref = np.array([o.rhs_point(yh, tuple(i)) for i in idx])
    got = np.array([bh[tuple(i)] for i in idx])
    scale = np.abs(bh).max()
    assert np.max(np.abs(got - ref)) <= 1e-12 * scale
    g32 = tca.Operator(A, L, c.lam, dtype="f32")
    b32 = g32.rhs(y.float()).cpu().numpy()
    got32 = np.array([b32[tuple(i)] for i in idx])
    assert np.max(np.abs(got32 - ref)) <= 1e-5 * scale
