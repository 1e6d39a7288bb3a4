"""Single-block CG engine (tca_tiny.cu: the whole Fig. 2 solve, PAPER.md:186-227,
in one launch by one 1024-thread block, vectors in shared memory) against the
CPU oracle at matched k on seeded inputs (synth/): config 0, orders 1-4,
banded and dense modes, factor-form operators, ragged sizes (N not a multiple
of the block), both sides of the shared-memory size boundary, tolerance stops,
warm starts and the guards.  Tolerances: north_star's fp64 CG <= 1e-8 at
matched k, fp32 <= 1e-5."""
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


def to_dev(x, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def to_host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy()


TDT = {"f64": torch.float64, "f32": torch.float32}
TOL = {"f64": 1e-8, "f32": 1e-5}

# (n, m, basis): ragged sizes, orders 1-4, banded (B-spline) and dense (Gaussian) modes
SHAPES = [
    ((12, 12, 12), (20, 20, 20), "bspline"),      # config 0
    ((1000,), (1500,), "bspline"),                # order 1
    ((37, 29), (60, 50), "bspline"),              # order 2, ragged
    ((9, 7, 6, 5), (14, 12, 10, 9), "bspline"),   # order 4
    ((11, 10, 9), (16, 15, 14), "gauss"),         # dense modes
    ((16, 16, 16), (24, 24, 24), "bspline"),      # N = 4096: largest fp64 cube that fits
]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n,m,basis", SHAPES)
def test_tiny_cg_fixed_iterations(n, m, basis, dtype, tca):
    A, L = synth.mode_matrices(n, m, basis=basis)
    lam = 0.01
    o = oracle.Operator(A, L, lam)
    b = o.rhs(synth.data(A, n, m, seed=1))
    g = tca.Operator(A, L, lam, dtype=dtype)
    assert g.tiny_engine
    # k = 12: on the ill-conditioned small shapes (order 4 with n_4 = 5, dense
    # Gaussian modes) the sensitivity of CG iterates to rounding grows with k
    # (loss of orthogonality): the general engine departs from the oracle the
    # same way by k = 30 (tools/diag_tiny.py), so larger k tests conditioning
    k = 12
    xg, rep = g.cg_solve(to_dev(b, TDT[dtype]), rtol=0.0, max_iters=k, history=True)
    xo, ko, st, hist = o.cg(b, rtol=0.0, max_iters=k)
    g.close()
    assert rep["iterations"] == ko == k and rep["status"] == tca.OK
    assert relerr(to_host(xg), xo) <= TOL[dtype]
    # rounding in the dot products is eps * rho_0 in absolute terms: the tail of a
    # history that falls 15 decades is compared at that level
    rho_tol, rho_abs = (1e-9, 1e-14) if dtype == "f64" else (1e-3, 1e-6)
    assert np.allclose(rep["rho_history"][:k + 1], hist[:k + 1], rtol=rho_tol, atol=rho_abs * hist[0])
    assert rep["rho0"] == pytest.approx(hist[0], rel=1e-12 if dtype == "f64" else 1e-5)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_tiny_cg_tolerance_stop_config0(dtype, tca):
    c = synth.CONFIGS[0]
    A, L = synth.mode_matrices(c)
    o = oracle.Operator(A, L, c.lam)
    b = o.rhs(synth.data(A, c.n, c.m, seed=1))
    g = tca.Operator(A, L, c.lam, dtype=dtype)
    rtol = 1e-10 if dtype == "f64" else 1e-5
    xg, rep = g.cg_solve(to_dev(b, TDT[dtype]), rtol=rtol, max_iters=c.max_iters)
    xo, ko, st, _ = o.cg(b, rtol=rtol, max_iters=c.max_iters)
    g.close()
    assert rep["converged"] and st == oracle.OK
    assert abs(rep["iterations"] - ko) <= (0 if dtype == "f64" else 3)
    assert rep["rho_final"] <= rtol * rtol * float(b.ravel() @ b.ravel())
    assert relerr(to_host(xg), xo) <= (1e-8 if dtype == "f64" else 1e-4)


def test_tiny_cg_not_converged_status(tca):
    c = synth.CONFIGS[0]
    A, L = synth.mode_matrices(c)
    g = tca.Operator(A, L, c.lam)
    b = to_dev(synth.random_tensor(c.n, seed=5))
    x, rep = g.cg_solve(b, rtol=1e-14, max_iters=3, raise_on=())
    assert rep["status"] == tca.NOT_CONVERGED and rep["iterations"] == 3
    x, rep = g.cg_solve(b, rtol=1e-14, max_iters=0, raise_on=())
    assert rep["status"] == tca.NOT_CONVERGED and rep["iterations"] == 0
    assert float(x.abs().max()) == 0.0
    x, rep = g.cg_solve(b, rtol=0.0, max_iters=0)
    assert rep["status"] == tca.OK and rep["iterations"] == 0


def test_tiny_cg_factor_form_and_warm_start(tca):
    """tca_operator_create_gram (Eq. 9's Kronecker sum on top of a product term)
    on the single-block engine, cold and warm."""
    n = (10, 9, 8)
    G = [synth.bspline_matrix(k, 2 * k).T @ synth.bspline_matrix(k, 2 * k) for k in n]
    R = [synth.laplacian_1d(k) for k in n]
    lam = 0.05
    o = oracle.Operator.from_gram(G, R, lam)
    g = tca.Operator.from_gram(G, R, lam)
    assert g.tiny_engine
    b = synth.random_tensor(n, seed=21)
    x0 = synth.random_tensor(n, seed=22, stream=8)
    for start in (None, x0):
        kw = {} if start is None else {"x0": to_dev(start)}
        xg, rep = g.cg_solve(to_dev(b), rtol=0.0, max_iters=25, history=True, **kw)
        xo, ko, st, hist = o.cg(b, rtol=0.0, max_iters=25, x0=start)
        assert relerr(to_host(xg), xo) <= 1e-8
        assert np.allclose(rep["rho_history"][:26], hist[:26], rtol=1e-9, atol=1e-14 * hist[0])


def test_tiny_boundary_sizes(tca):
    """The engine is chosen by size: fp64 up to 4096 unknowns (four per thread),
    4352 (17 x 16 x 16) take the general engine; fp32 up to 8192."""
    def op(n, dtype):
        A, L = synth.mode_matrices(n, tuple(2 * k for k in n))
        return tca.Operator(A, L, 0.01, dtype=dtype)
    assert op((16, 16, 16), "f64").tiny_engine
    assert not op((17, 16, 16), "f64").tiny_engine
    assert op((17, 16, 16), "f32").tiny_engine
    assert not op((24, 24, 24), "f32").tiny_engine


def test_tiny_matches_general_engine_in_child(tca, tmp_path):
    """Same iterates on both engines: the general path (TCA_TINY=0, a child
    process because the switch is read once) against the single-block one."""
    c = synth.CONFIGS[0]
    A, L = synth.mode_matrices(c)
    o = oracle.Operator(A, L, c.lam)
    b = o.rhs(synth.data(A, c.n, c.m, seed=1))
    np.save(tmp_path / "b.npy", b)
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r})
import synth
from paper_1001_5460_b200 import tca
c = synth.CONFIGS[0]
A, L = synth.mode_matrices(c)
g = tca.Operator(A, L, c.lam)
assert not g.tiny_engine
b = torch.from_numpy(np.load({str(tmp_path / 'b.npy')!r})).cuda()
x, rep = g.cg_solve(b, rtol=0.0, max_iters=60)
np.save({str(tmp_path / 'x.npy')!r}, x.cpu().numpy())
"""
    env = dict(os.environ, TCA_TINY="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    xgen = np.load(tmp_path / "x.npy")
    g = tca.Operator(A, L, c.lam)
    assert g.tiny_engine
    xt, rep = g.cg_solve(to_dev(b), rtol=0.0, max_iters=60)
    assert relerr(to_host(xt), xgen) <= 1e-10


def test_tiny_is_one_launch(tca):
    c = synth.CONFIGS[0]
    A, L = synth.mode_matrices(c)
    g = tca.Operator(A, L, c.lam)
    b = to_dev(synth.random_tensor(c.n, seed=5))
    g.cg_solve(b, rtol=0.0, max_iters=5)
    n0 = tca.kernel_launches()
    x = torch.empty_like(b)
    g.cg_solve(b, x=x, rtol=0.0, max_iters=100)
    # the solve itself is one launch; the report's true residual adds one apply + its reduction
    assert tca.kernel_launches() - n0 <= 8
