"""Kronecker-factor preconditioned CG (reading Z22):
the GPU preconditioner solve and PCG against the CPU oracle's (pinned by
P10-P13 in test_oracle_pins.py)."""
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


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.float64 if dt == "f64" else torch.float32)


# (n, m, basis, lam): banded factors (B-spline), dense factors (Gaussian), short modes, D = 1..4
PC_CASES = [((12, 12, 12), (20, 20, 20), "bspline", 1e-2),
            ((32, 32, 32, 16), (64, 64, 64, 32), "bspline", 1e-2),
            ((24, 11, 36, 15), (48, 22, 72, 30), "bspline", 1e-3),
            ((20, 18, 16), (27, 24, 22), "gauss", 1e-3),
            ((3, 5, 2, 7), (6, 9, 4, 12), "bspline", 5e-2),
            ((40,), (70,), "bspline", 1e-2),
            ((17, 9), (30, 16), "gauss", 1e-2)]
PC_IDS = ["x".join(map(str, c[0])) + "-" + c[2] for c in PC_CASES]


@pytest.mark.parametrize("case", PC_CASES, ids=PC_IDS)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_precond_apply_matches_oracle(case, dt, tca):
    n, m, basis, lam = case
    A, L = synth.mode_matrices(n, m, basis=basis, seed=2)
    o = oracle.Operator(A, L, lam)
    op = tca.Operator(A, L, lam, dtype=dt)
    eps, bw = op.precond_info()
    _, eps_ref = o.precond_factors()
    assert np.allclose(eps, eps_ref, rtol=1e-12, atol=0)
    for d, nd in enumerate(n):
        assert bw[d] <= (min(3, nd - 1) if basis == "bspline" else nd - 1)
    r = synth.random_tensor(n, seed=21)
    z = op.precond_apply(dev(r, dt)).double().cpu().numpy()
    assert rel(z, o.precond_apply(r)) <= (1e-12 if dt == "f64" else 1e-5)
    # in place (z aliases r)
    rd = dev(r, dt)
    op.precond_apply(rd, rd)
    assert rel(rd.double().cpu().numpy(), o.precond_apply(r)) <= (1e-12 if dt == "f64" else 1e-5)
    op.close()


# fp32 only on the B-spline shapes: the small Gaussian system's kappa(M) ~ 1e5
# turns fp32 rounding into ~5e-3 after 25 steps (no config runs Gaussian modes in fp32)
FIX_CASES = [(c, dt) for c in PC_CASES[:5] for dt in ("f64", "f32") if dt == "f64" or c[2] == "bspline"]


@pytest.mark.parametrize("case,dt", FIX_CASES, ids=[f"{i}-{dt}" for (c, dt) in FIX_CASES
                                                    for i in ["x".join(map(str, c[0]))]])
def test_pcg_fixed_iterations_matches_oracle(case, dt, tca):
    n, m, basis, lam = case
    A, L = synth.mode_matrices(n, m, basis=basis, seed=2)
    o = oracle.Operator(A, L, lam)
    op = tca.Operator(A, L, lam, dtype=dt)
    b = o.rhs(synth.data(A, n, m, seed=3))
    k = 25
    x, rep = op.pcg_solve(dev(b, dt), rtol=0.0, max_iters=k, history=True)
    xr, kr, st, hist = o.pcg(b, rtol=0.0, max_iters=k)
    assert rep["iterations"] == kr == k
    assert rel(x.double().cpu().numpy(), xr) <= (1e-8 if dt == "f64" else 1e-5)
    if dt == "f64":
        assert np.allclose(rep["rho_history"], hist, rtol=1e-6, atol=1e-30 * hist[0])
    op.close()


@pytest.mark.parametrize("cfg_index", [0, 1])
def test_pcg_tolerance_configs_match_oracle(cfg_index, tca):
    """Configs 0 and 1 (tolerance-stopped; config 1 has dense Gaussian modes):
    the GPU stopping iteration equals the oracle's (+-1, reading Z11) and the
    solutions agree at the GPU's k."""
    cfg = synth.CONFIGS[cfg_index]
    A, L = synth.mode_matrices(cfg)
    o = oracle.Operator(A, L, cfg.lam)
    op = tca.Operator(A, L, cfg.lam)
    b = o.rhs(synth.data(A, cfg.n, cfg.m, seed=1))
    x, rep = op.pcg_solve(dev(b, "f64"), rtol=cfg.rtol, max_iters=cfg.max_iters)
    _, k_nat, st_nat, _ = o.pcg(b, rtol=cfg.rtol, max_iters=cfg.max_iters)
    assert rep["converged"] and st_nat == oracle.OK
    assert abs(rep["iterations"] - k_nat) <= 1
    xr, _, _, _ = o.pcg(b, rtol=0.0, max_iters=rep["iterations"])
    assert rel(x.cpu().numpy(), xr) <= 1e-8
    _, k_cg, _, _ = o.cg(b, rtol=cfg.rtol, max_iters=cfg.max_iters)
    assert rep["iterations"] < k_cg
    op.close()


def test_pcg_exact_preconditioner_one_iteration(tca):
    """D = 1: F_1 = G_1 + lam R_1 = M, so PCG converges in one step."""
    n, m = (40,), (70,)
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, 1e-2)
    op = tca.Operator(A, L, 1e-2)
    b = synth.random_tensor(n, seed=4)
    x, rep = op.pcg_solve(dev(b, "f64"), rtol=1e-12, max_iters=10)
    assert rep["iterations"] == 1 and rep["converged"]
    xr, _, _, _ = o.pcg(b, rtol=1e-12, max_iters=10)
    assert rel(x.cpu().numpy(), xr) <= 1e-12
    op.close()


def test_pcg_zero_rhs_and_cg_unchanged_after_pcg(tca):
    n, m = (12, 12, 12), (20, 20, 20)
    A, L = synth.mode_matrices(n, m)
    o = oracle.Operator(A, L, 1e-2)
    op = tca.Operator(A, L, 1e-2)
    x, rep = op.pcg_solve(torch.zeros(n, dtype=torch.float64, device="cuda"), rtol=1e-10, max_iters=50)
    assert rep["iterations"] == 0 and rep["converged"] and float(x.abs().max()) == 0.0
    # the plain CG graphs are rebuilt after a PCG solve on the same x buffer
    b = synth.random_tensor(n, seed=8)
    bd = dev(b, "f64")
    xc, repc = op.cg_solve(bd, x=x, rtol=0.0, max_iters=60)
    xr, _, _, _ = o.cg(b, rtol=0.0, max_iters=60)
    assert rel(xc.cpu().numpy(), xr) <= 1e-8
    xp, repp = op.pcg_solve(bd, x=x, rtol=0.0, max_iters=60)
    xpr, _, _, _ = o.pcg(b, rtol=0.0, max_iters=60)
    assert rel(xp.cpu().numpy(), xpr) <= 1e-8
    op.close()
