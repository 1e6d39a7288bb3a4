"""GPU parity at the headline sizes and for the solver boundary (C ABI) against
the CPU oracle on identical seeded inputs (synth/).  Tolerances are
BASELINE.json north_star's: fp64 apply <= 1e-12 relative L2, CG <= 1e-8 at
matched iteration count, fp32 <= 1e-5 (against the fp64 oracle).

  * config 3 (128^3 x 15, the bench workload): the whole apply output, and the
    500-iteration CG of the bench (fp64 and the default fp32 path) at matched
    k with the first 20 rho values (Fig. 2);
  * config 4 (256^3 x 32, 537 M unknowns): three CG iterations on the full
    tensor;
  * the warm start x0_zero = 0 (Fig. 2's R := B - A*C) for
    CG, PCG and single-reduction CG, relres_final (reading Z2), the
    breakdown and non-finite guards, and tca_solve_host_batch with a
    tolerance stop that some items miss."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


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


# ------------------------------------------------------------------ config 3, whole tensors
@pytest.fixture(scope="module")
def cfg3():
    c = synth.CONFIGS[3]
    A, L = synth.mode_matrices(c)
    o = oracle.Operator(A, L, c.lam)
    return c, A, L, o


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_cfg3_apply_whole_tensor(dtype, tol, tca, cfg3):
    c, A, L, o = cfg3
    x = synth.random_tensor(c.n, seed=9)
    g = tca.Operator(A, L, c.lam, dtype=dtype)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    y = to_host(g.apply(to_dev(x, tdt)))
    g.close()
    assert relerr(y, o.apply(x)) <= tol


@pytest.fixture(scope="module")
def cfg3_cg_oracle(cfg3):
    """The bench's solve: b = (kron A_d^T) y for the seeded synthetic data, 500
    Fig. 2 iterations from x0 = 0 in the oracle (minutes on the host cores)."""
    c, A, L, o = cfg3
    b = o.rhs(synth.data(A, c.n, c.m, seed=1))
    xo, ko, st, hist = o.cg(b, rtol=0.0, max_iters=c.max_iters)
    assert ko == c.max_iters and st == oracle.OK
    return b, xo, hist


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-8), ("f32", 1e-5)])
def test_cfg3_cg_500_iterations_against_oracle(dtype, tol, tca, cfg3, cfg3_cg_oracle):
    c, A, L, o = cfg3
    b, xo, hist = cfg3_cg_oracle
    g = tca.Operator(A, L, c.lam, dtype=dtype)
    assert g.apply_path == "fused"
    tdt = torch.float64 if dtype == "f64" else torch.float32
    xg, rep = g.cg_solve(to_dev(b, tdt), rtol=0.0, max_iters=c.max_iters, history=True)
    g.close()
    assert rep["iterations"] == c.max_iters
    assert relerr(to_host(xg), xo) <= tol
    rho_tol = 1e-10 if dtype == "f64" else 1e-4
    assert np.allclose(rep["rho_history"][:20], hist[:20], rtol=rho_tol, atol=0.0)


# ------------------------------------------------------------------ config 4, whole tensor, k = 3
def test_cfg4_cg_three_iterations_whole_tensor(tca):
    c = synth.CONFIGS[4]
    A, L = synth.mode_matrices(c)
    b = synth.random_tensor(c.n, seed=13)
    g = tca.Operator(A, L, c.lam)
    assert g.apply_path == "fused"
    xg, rep = g.cg_solve(to_dev(b), rtol=0.0, max_iters=3, history=True)
    xh = to_host(xg)
    del xg
    g.close()
    torch.cuda.empty_cache()
    o = oracle.Operator(A, L, c.lam)
    xo, ko, st, hist = o.cg(b, rtol=0.0, max_iters=3)
    assert ko == 3 and rep["iterations"] == 3
    assert relerr(xh, xo) <= 1e-8
    assert np.allclose(rep["rho_history"], hist, rtol=1e-10, atol=0.0)


# ------------------------------------------------------------------ warm start, true residual
WARM_CASES = [(0, "cg"), (2, "cg"), (2, "pcg"), (2, "cgsr"), (0, "cgsr")]


@pytest.mark.parametrize("cfg,solver", WARM_CASES)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_warm_start_matches_oracle_at_matched_k(cfg, solver, dtype, tca):
    c = synth.CONFIGS[cfg]
    A, L = synth.mode_matrices(c)
    o = oracle.Operator(A, L, c.lam)
    b = o.rhs(synth.data(A, c.n, c.m, seed=1))
    x0 = synth.random_tensor(c.n, seed=41, stream=8)
    g = tca.Operator(A, L, c.lam, dtype=dtype)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    k = 15
    xg, rep = getattr(g, solver + "_solve")(to_dev(b, tdt), rtol=0.0, max_iters=k, x0=to_dev(x0, tdt),
                                            history=True)
    xo, ko, st, hist = getattr(o, solver)(b, rtol=0.0, max_iters=k, x0=x0)
    assert rep["iterations"] == ko == k
    tol = 1e-8 if dtype == "f64" else 1e-5
    assert relerr(to_host(xg), xo) <= tol
    # rho_0 = <B - A C, B - A C> of the warm start
    assert abs(rep["rho0"] - hist[0]) <= (1e-10 if dtype == "f64" else 1e-5) * hist[0]
    # the report's true residual |b - M x_k| / |b|
    res = relerr(o.apply(to_host(xg)), b)
    assert abs(rep["relres_final"] - res) <= (1e-6 if dtype == "f64" else 1e-3) * res + 1e-15


def test_warm_start_tolerance_stop_is_relative_to_b(tca):
    """Reading Z28: the stop reference is <b, b>; a start at the solution stops
    within one iteration, a poor start runs to the same relative residual."""
    c = synth.CONFIGS[2]
    A, L = synth.mode_matrices(c)
    o = oracle.Operator(A, L, c.lam)
    b = o.rhs(synth.data(A, c.n, c.m, seed=1))
    g = tca.Operator(A, L, c.lam)
    xs, rep = g.cg_solve(to_dev(b), rtol=1e-12, max_iters=400)
    assert rep["converged"] and rep["relres_final"] <= 1e-10
    x1, rep1 = g.cg_solve(to_dev(b), rtol=1e-8, max_iters=400, x0=xs)
    assert rep1["converged"] and rep1["iterations"] <= 1
    x0 = 10.0 * synth.random_tensor(c.n, seed=42, stream=8)
    x2, rep2 = g.cg_solve(to_dev(b), rtol=1e-10, max_iters=400, x0=to_dev(x0))
    assert rep2["converged"] and rep2["rho_final"] <= 1e-20 * float(b.ravel() @ b.ravel())
    xo, ko, _, _ = o.cg(b, rtol=1e-10, max_iters=400, x0=x0)
    assert abs(ko - rep2["iterations"]) <= 1
    assert relerr(to_host(x2), to_host(xs)) <= 1e-8


def test_relres_final_cold_start(tca):
    c = synth.CONFIGS[0]
    A, L = synth.mode_matrices(c)
    o = oracle.Operator(A, L, c.lam)
    b = o.rhs(synth.data(A, c.n, c.m, seed=1))
    g = tca.Operator(A, L, c.lam)
    for iters in (3, 20):
        xg, rep = g.cg_solve(to_dev(b), rtol=0.0, max_iters=iters)
        res = relerr(o.apply(to_host(xg)), b)
        assert abs(rep["relres_final"] - res) <= 1e-6 * res
    xg, rep = g.cg_solve(torch.zeros(c.n, dtype=torch.float64, device="cuda"), rtol=1e-10, max_iters=5)
    assert rep["relres_final"] == 0.0


# ------------------------------------------------------------------ device guards
def test_breakdown_guard_on_indefinite_operator(tca):
    """<p, Mp> <= 0 stops with TCA_ERR_BREAKDOWN: M = G + lambda R
    built from factors with R = -I (indefinite for lambda = 5)."""
    n = (8, 6, 5)
    G = [synth.bspline_matrix(k, 2 * k).T @ synth.bspline_matrix(k, 2 * k) for k in n]
    R = [-np.eye(k) for k in n]
    g = tca.Operator.from_gram(G, R, 5.0)
    b = to_dev(synth.random_tensor(n, seed=43))
    for solver in ("cg_solve", "cgsr_solve"):
        x, rep = getattr(g, solver)(b, rtol=1e-10, max_iters=50, raise_on=())
        assert rep["status"] == tca.ERR_BREAKDOWN
        assert rep["iterations"] <= 1
        assert np.isfinite(to_host(x)).all()
    with pytest.raises(tca.TcaError) as ei:
        g.cg_solve(b, rtol=1e-10, max_iters=50)
    assert ei.value.status == tca.ERR_BREAKDOWN


def test_nonfinite_guard(tca):
    c = synth.CONFIGS[0]
    A, L = synth.mode_matrices(c)
    g = tca.Operator(A, L, c.lam)
    b = synth.random_tensor(c.n, seed=44)
    b[3, 4, 5] = np.nan
    for solver in ("cg_solve", "pcg_solve", "cgsr_solve"):
        x, rep = getattr(g, solver)(to_dev(b), rtol=1e-10, max_iters=20, raise_on=())
        assert rep["status"] == tca.ERR_NONFINITE
        assert rep["iterations"] == 0
    b[3, 4, 5] = np.inf
    with pytest.raises(tca.TcaError) as ei:
        g.cg_solve(to_dev(b), rtol=0.0, max_iters=5)
    assert ei.value.status == tca.ERR_NONFINITE


# ------------------------------------------------------------------ host batch with a tolerance stop
def test_solve_host_batch_not_converged_items_all_written(tca):
    """an item that misses rtol must not stop the batch; every x_host[i]
    equals its single solve and the call returns TCA_NOT_CONVERGED."""
    c = synth.CONFIGS[2]
    A, L = synth.mode_matrices(c)
    g = tca.Operator(A, L, c.lam)
    ys = [torch.from_numpy(synth.data(A, c.n, c.m, seed=s)).pin_memory() for s in (1, 2, 3)]
    xs = [torch.zeros(c.n, dtype=torch.float64).pin_memory() for _ in ys]
    reps = g.solve_host_batch(ys, xs, rtol=1e-12, max_iters=7)
    assert all(r["status"] == tca.NOT_CONVERGED and r["iterations"] == 7 for r in reps)
    for y, x in zip(ys, xs):
        b = g.rhs(y.cuda())
        xr, _ = g.cg_solve(b, rtol=1e-12, max_iters=7, raise_on=())
        assert torch.equal(x, xr.cpu())
