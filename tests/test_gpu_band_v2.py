"""GPU parity of the opt-in warp-specialised fused apply (tca_band2.cuh,
TCA_BAND_V2=1).  The switch is read once per process, so the
checks run in a child interpreter.  Same tolerances as test_gpu_parity.py
(north_star: fp64 apply <= 1e-12, CG <= 1e-8 at matched k, fp32 <= 1e-5)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import numpy as np, torch
import oracle, synth
from paper_1001_5460_b200 import tca
def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))
cases = [((32, 32, 32, 16), (64, 64, 64, 32), 1e-2),   # config 2
         ((13, 11, 36, 15), (26, 22, 72, 30), 1e-3),   # ragged tiles, n4 = 15
         ((40, 30, 48, 15), (80, 60, 96, 30), 1e-2)]   # several tiles per CTA
for n, m, lam in cases:
    A, L = synth.mode_matrices(n, m, basis="bspline", seed=1)
    o = oracle.Operator(A, L, lam)
    x = synth.random_tensor(n, seed=5)
    ref = o.apply(x)
    for dt, tol in (("f64", 1e-12), ("f32", 1e-5)):
        g = tca.Operator(A, L, lam, dtype=dt)
        assert g.apply_path == "fused"
        tdt = torch.float64 if dt == "f64" else torch.float32
        y = g.apply(torch.from_numpy(x).to("cuda", tdt)).double().cpu().numpy()
        e = rel(y, ref)
        assert e <= tol, (n, dt, e)
    # CG (the <p, q> epilogue) against the oracle at matched k
    b = synth.random_tensor(n, seed=7)
    g = tca.Operator(A, L, lam, dtype="f64")
    xg, rep = g.cg_solve(torch.from_numpy(b).cuda(), rtol=0.0, max_iters=25)
    xo, _, _, _ = o.cg(b, rtol=0.0, max_iters=25)
    e = rel(xg.cpu().numpy(), xo)
    assert e <= 1e-8, (n, "cg", e)
print("band v2 parity ok")
"""


def test_band_v2_parity_child_process():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, TCA_BAND_V2="1", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "band v2 parity ok" in r.stdout
