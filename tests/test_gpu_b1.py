"""Fused CG step B1' (one kernel reads R|Z, P_old and C and
writes P_new, C and Q = M P_new with <P_new, Q>, opt-in with
TCA_B1=1): CG and PCG iterates against the CPU oracle's Fig. 2 (CG <= 1e-8 at
matched k, fp32 <= 1e-5), and against the default unfused step on the same inputs."""
import os

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


def dev(a, dt="f64"):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.float64 if dt == "f64" else torch.float32)


def make_op(tca, A, L, lam, dt, b1=True):
    """Operator whose first solve decides the step: fused with TCA_B1=1, else unfused."""
    return tca.Operator(A, L, lam, dtype=dt)


def solve(op, b, dt, b1, how="cg", **kw):
    # the general (graph-chunked) engine: the single-block and grid engines take
    # small shapes otherwise, and B1' is a step of the general engine only
    env = {"TCA_GRID": "0", "TCA_TINY": "0"}
    if b1:
        env["TCA_B1"] = "1"
    os.environ.update(env)
    try:
        fn = op.cg_solve if how == "cg" else op.pcg_solve
        return fn(dev(b, dt), **kw)
    finally:
        for k in env:
            os.environ.pop(k, None)


def expect_b1(n, dt):
    """B1' needs the parameter-block tap tables and the unpadded staging layout:
    a mode-4 fibre that is a multiple of 32 B (fp64 n4 = 4, 8, 16, 32; fp32 n4 =
    8, 16, 32) is staged with a padded fibre pitch (Cfg::PADDED),
    which B1' does not take (unfused)."""
    n4 = n[3] if len(n) == 4 else 1
    es = 8 if dt == "f64" else 4
    return (n4 * es) % 32 != 0


# fused-path shapes: ragged mode-2/3 tiles (clipped stores), every n4 class, a
# tile grid larger than the persistent grid (split schedule), D = 3
B1_CASES = [((32, 32, 30, 15), (64, 64, 60, 30), 1e-2),
            ((13, 11, 36, 15), (26, 22, 72, 30), 1e-3),
            ((32, 32, 32, 16), (64, 64, 64, 32), 1e-2),
            ((40, 30, 48, 15), (80, 60, 96, 30), 1e-2),
            ((9, 70, 16, 7), (18, 140, 32, 14), 0.5),
            ((7, 9, 33, 8), (14, 18, 66, 16), 1e-2),
            ((11, 6, 21, 4), (22, 12, 42, 8), 1e-2),
            ((6, 20, 20, 32), (9, 30, 30, 48), 1e-3),
            ((14, 13, 12), (28, 26, 24), 1e-2),
            ((5, 100, 160, 1), (8, 150, 240, 2), 1e-2),
            ((4, 200, 112, 15), (8, 400, 224, 30), 1e-2)]   # 350 tiles > 320 CTAs: split schedule
B1_IDS = ["x".join(map(str, c[0])) for c in B1_CASES]


@pytest.mark.parametrize("case", B1_CASES, ids=B1_IDS)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_b1_cg_fixed_iterations_match_oracle(case, dt, tca):
    n, m, lam = case
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    b = o.rhs(synth.data(A, n, m, seed=3))
    # f64: > one graph chunk (32): eager first step, one replay, eager tail.
    # fp32: 20 steps (fp32 rounding grows with k on the ill-conditioned small shapes)
    k = 45 if dt == "f64" else 20
    op = make_op(tca, A, L, lam, dt)
    x, rep = solve(op, b, dt, True, rtol=0.0, max_iters=k, history=True)
    assert op.cg_fused_step is (op.apply_path == "fused" and expect_b1(n, dt))
    xr, kr, _, hist = o.cg(b, rtol=0.0, max_iters=k)
    assert rep["iterations"] == kr == k
    assert rel(x.double().cpu().numpy(), xr) <= (1e-8 if dt == "f64" else 1e-5)
    if dt == "f64":
        assert np.allclose(rep["rho_history"][:20], hist[:20], rtol=1e-6)
    op.close()


@pytest.mark.parametrize("case", B1_CASES[:3], ids=B1_IDS[:3])
def test_b1_matches_unfused_step(case, tca):
    n, m, lam = case
    A, L = synth.mode_matrices(n, m, seed=2)
    b = oracle.Operator(A, L, lam).rhs(synth.data(A, n, m, seed=3))
    res = []
    for b1 in (True, False):
        op = make_op(tca, A, L, lam, "f64", b1)
        x, rep = solve(op, b, "f64", b1, rtol=0.0, max_iters=70, history=True)
        assert op.cg_fused_step is (b1 and expect_b1(n, "f64"))
        res.append((x.cpu().numpy(), rep))
        op.close()
    (x1, r1), (x0, r0) = res
    assert r1["iterations"] == r0["iterations"] == 70
    assert rel(x1, x0) <= 1e-10   # same arithmetic per element; <P, Q> summed per CTA differently
    assert np.allclose(r1["rho_history"][:30], r0["rho_history"][:30], rtol=1e-9)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_b1_tolerance_stop_mid_chunk(dt, tca):
    """Convergence inside a graph chunk: later steps only apply the pending C update
    (device done flag), so x is exactly the oracle's x_k at the GPU's k."""
    n, m, lam = (12, 12, 12), (20, 20, 20), 1e-2
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    b = o.rhs(synth.data(A, n, m, seed=1))
    op = make_op(tca, A, L, lam, dt)
    rtol = 1e-10 if dt == "f64" else 1e-5
    x, rep = solve(op, b, dt, True, rtol=rtol, max_iters=500)
    assert op.cg_fused_step is True and rep["converged"]
    _, k_nat, _, _ = o.cg(b, rtol=rtol, max_iters=500)
    assert abs(rep["iterations"] - k_nat) <= 1
    xr, _, _, _ = o.cg(b, rtol=0.0, max_iters=rep["iterations"])
    assert rel(x.double().cpu().numpy(), xr) <= (1e-8 if dt == "f64" else 1e-5)
    op.close()


def test_b1_pcg_matches_oracle(tca):
    n, m, lam = (24, 11, 36, 15), (48, 22, 72, 30), 1e-3
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    b = o.rhs(synth.data(A, n, m, seed=3))
    op = make_op(tca, A, L, lam, "f64")
    x, rep = solve(op, b, "f64", True, how="pcg", rtol=0.0, max_iters=40, history=True)
    assert op.cg_fused_step is True
    xr, kr, _, hist = o.pcg(b, rtol=0.0, max_iters=40)
    assert rep["iterations"] == kr == 40
    assert rel(x.cpu().numpy(), xr) <= 1e-8
    assert np.allclose(rep["rho_history"], hist, rtol=1e-6, atol=1e-30 * hist[0])
    op.close()


def test_b1_repeated_solves_and_x_reuse(tca):
    """The P ping-pong restarts at every solve; cached graphs stay valid."""
    n, m, lam = (32, 32, 30, 15), (64, 64, 60, 30), 1e-2
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    op = make_op(tca, A, L, lam, "f64")
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    for seed, k in ((3, 33), (4, 64), (5, 7)):
        b = synth.random_tensor(n, seed=seed)
        xg, rep = solve(op, b, "f64", True, x=x, rtol=0.0, max_iters=k)
        assert op.cg_fused_step is True
        xr, _, _, _ = o.cg(b, rtol=0.0, max_iters=k)
        assert rep["iterations"] == k
        assert rel(xg.cpu().numpy(), xr) <= 1e-8
    op.close()


def test_b1_full_size_cfg3_residual_sampled(tca):
    """Config 3 (the bench workload, whole-tile schedule): 500 B1' steps, then
    M x = b on sampled rows by the oracle's point evaluation."""
    c = synth.CONFIGS[3]
    A, L = synth.mode_matrices(c)
    g = tca.Operator(A, L, c.lam)
    b = synth.random_tensor(c.n, seed=9)
    xg, rep = solve(g, b, "f64", True, rtol=0.0, max_iters=c.max_iters)
    assert g.cg_fused_step is True and rep["iterations"] == c.max_iters
    xh = xg.cpu().numpy()
    o = oracle.Operator(A, L, c.lam)
    rng = np.random.default_rng(1)
    pts = [tuple(int(rng.integers(0, nd)) for nd in c.n) for _ in range(100)]
    pts += [(0, 0, 0, 0), tuple(nd - 1 for nd in c.n), (127, 0, 64, 7), (2, 127, 126, 0)]
    Mx = o.apply_points(xh, pts)
    bb = np.array([b[p] for p in pts])
    assert np.max(np.abs(Mx - bb)) <= 1e-6 * np.abs(b).max()
    g.close()


@pytest.mark.parametrize("k", [1, 2, 8, 32, 33])
def test_b1_short_solves(k, tca):
    """Fewer steps than a graph chunk (chunks captured but not replayed: every
    tensor map must already be on the device), and the chunk boundaries."""
    n, m, lam = (32, 32, 30, 15), (64, 64, 60, 30), 1e-2
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    b = synth.random_tensor(n, seed=6)
    op = make_op(tca, A, L, lam, "f64")
    x, rep = solve(op, b, "f64", True, rtol=0.0, max_iters=k)
    assert op.cg_fused_step is True and rep["iterations"] == k
    xr, _, _, _ = o.cg(b, rtol=0.0, max_iters=k)
    assert rel(x.cpu().numpy(), xr) <= 1e-8
    op.close()


# ------------------------------------------------------------------ pipelined host solves
def test_solve_host_batch_matches_single_solves(tca):
    """tca_solve_host_batch: every item equals its own tca_solve_host (same
    kernels and reductions) and the oracle's Fig. 2 iterate; copies of
    neighbouring items overlap the compute (odd count: both buffer parities)."""
    n, m, lam = (16, 12, 20, 15), (32, 24, 40, 30), 1e-2
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    op = tca.Operator(A, L, lam)
    ys = [torch.from_numpy(synth.data(A, n, m, seed=s)).contiguous().pin_memory() for s in (3, 4, 5)]
    xs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in ys]
    reps = op.solve_host_batch(ys, xs, rtol=0.0, max_iters=40)
    assert [r["iterations"] for r in reps] == [40, 40, 40]
    for y, x in zip(ys, xs):
        x1 = torch.empty(n, dtype=torch.float64).pin_memory()
        op.solve_host(y, x1, rtol=0.0, max_iters=40)
        assert torch.equal(x, x1)
        xr, _, _, _ = o.cg(o.rhs(y.numpy()), rtol=0.0, max_iters=40)
        assert rel(x.numpy(), xr) <= 1e-8
    assert op.solve_host_batch([], [], max_iters=5) == []
    op.close()
