"""Deferred x update (include/tca.h tca_operator_cg_deferred_x):
the x update of Fig. 2 (C := C + alpha P) runs one iteration
late, streamed by an extra warp of the next banded apply, with P_next formed
into a second P buffer.  Same arithmetic per element as the three-kernel
iteration, so the iterates match it bit for bit; against the CPU oracle's
Fig. 2 at matched k (fp64 <= 1e-8, fp32 <= 1e-5), across graph-chunk
boundaries, tolerance stops inside a chunk (the pending update of the last
iteration), repeated solves and PCG."""
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


def dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.float64 if dt == "f64" else torch.float32)


GENERAL = {"TCA_GRID": "0", "TCA_TINY": "0"}   # the general (graph-chunked) engine on small shapes


def solve(op, b, dt, dx, how="cg", **kw):
    """First solve of `op` decides the step: TCA_DX=1 forces the deferred update, 0 turns it off."""
    env = dict(GENERAL, TCA_DX="1" if dx else "0")
    os.environ.update(env)
    try:
        assert op.cg_engine == "general"
        fn = op.cg_solve if how == "cg" else op.pcg_solve
        return fn(dev(b, dt), **kw)
    finally:
        for k in env:
            os.environ.pop(k, None)


CASES = [((32, 32, 30, 15), (64, 64, 60, 30), 1e-2),
         ((13, 11, 36, 15), (26, 22, 72, 30), 1e-3),
         ((7, 9, 33, 8), (14, 18, 66, 16), 1e-2),
         ((14, 13, 12), (28, 26, 24), 1e-2),
         ((6, 20, 20, 32), (9, 30, 30, 48), 1e-3)]
IDS = ["x".join(map(str, c[0])) for c in CASES]


@pytest.mark.parametrize("case", CASES, ids=IDS)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_dx_matches_oracle_and_three_kernel_step(case, dt, tca):
    n, m, lam = case
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    b = o.rhs(synth.data(A, n, m, seed=3))
    k = 45 if dt == "f64" else 20   # > one graph chunk (32) in fp64
    res = []
    for dx in (True, False):
        op = tca.Operator(A, L, lam, dtype=dt)
        x, rep = solve(op, b, dt, dx, rtol=0.0, max_iters=k, history=True)
        assert op.cg_deferred_x is (dx and op.apply_path == "fused")
        assert rep["iterations"] == k
        res.append((x.double().cpu().numpy(), rep))
        op.close()
    (x1, r1), (x0, r0) = res
    # same arithmetic per element; <P, Q> is summed over a different CTA partition
    # (the mode-1-synchronous schedule), so alpha may differ in the last bit
    assert rel(x1, x0) <= (1e-10 if dt == "f64" else 1e-6)
    assert np.allclose(r1["rho_history"][:30], r0["rho_history"][:30], rtol=1e-9 if dt == "f64" else 1e-5)
    xr, kr, _, hist = o.cg(b, rtol=0.0, max_iters=k)
    assert rel(x1, xr) <= (1e-8 if dt == "f64" else 1e-5)
    if dt == "f64":
        assert np.allclose(r1["rho_history"][:20], hist[:20], rtol=1e-6)


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("k", [1, 2, 31, 32, 33, 64, 65])
def test_dx_iteration_counts(dt, k, tca):
    """Solves shorter than, equal to and across graph chunks: the pending update of
    the last iteration is applied after the loop."""
    n, m, lam = (32, 32, 32, 15), (64, 64, 64, 30), 1e-2   # fused in both dtypes (n3 n4 esize % 16 == 0)
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    b = synth.random_tensor(n, seed=6)
    op = tca.Operator(A, L, lam, dtype=dt)
    x, rep = solve(op, b, dt, True, rtol=0.0, max_iters=k)
    assert op.cg_deferred_x is True and rep["iterations"] == k
    xr, _, _, _ = o.cg(b, rtol=0.0, max_iters=k)
    assert rel(x.double().cpu().numpy(), xr) <= (1e-8 if dt == "f64" else 2e-5)
    op.close()


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_dx_tolerance_stop_mid_chunk(dt, tca):
    """Convergence inside a graph chunk: the next apply applies only the pending
    x update (device done flag) and later ones nothing, so x is the oracle's x_k."""
    n, m, lam = (20, 22, 16, 15), (40, 44, 32, 30), 1e-2
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    b = o.rhs(synth.data(A, n, m, seed=1))
    rtol = 1e-10 if dt == "f64" else 1e-5
    op = tca.Operator(A, L, lam, dtype=dt)
    x, rep = solve(op, b, dt, True, rtol=rtol, max_iters=500)
    assert op.cg_deferred_x is True and rep["converged"]
    xr, _, _, _ = o.cg(b, rtol=0.0, max_iters=rep["iterations"])
    assert rel(x.double().cpu().numpy(), xr) <= (1e-8 if dt == "f64" else 1e-5)
    assert rep["relres_final"] <= (1e-8 if dt == "f64" else 1e-3)
    op.close()


def test_dx_pcg_and_warm_start(tca):
    n, m, lam = (24, 11, 36, 15), (48, 22, 72, 30), 1e-3
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    b = o.rhs(synth.data(A, n, m, seed=3))
    op = tca.Operator(A, L, lam, dtype="f64")
    x, rep = solve(op, b, "f64", True, how="pcg", rtol=0.0, max_iters=40, history=True)
    assert op.cg_deferred_x is True
    xr, kr, _, hist = o.pcg(b, rtol=0.0, max_iters=40)
    assert rep["iterations"] == kr == 40
    assert rel(x.cpu().numpy(), xr) <= 1e-8
    assert np.allclose(rep["rho_history"], hist, rtol=1e-6, atol=1e-30 * hist[0])
    # warm start from the PCG result: R := B - A*C, then CG (same operator, deferred x)
    x0 = synth.random_tensor(n, seed=11)
    os.environ.update(GENERAL)
    try:
        xw, repw = op.cg_solve(dev(b, "f64"), x0=dev(x0, "f64"), rtol=0.0, max_iters=37)
    finally:
        for kk in GENERAL:
            os.environ.pop(kk, None)
    xo, _, _, _ = o.cg(b, rtol=0.0, max_iters=37, x0=x0)
    assert rel(xw.cpu().numpy(), xo) <= 1e-8
    op.close()


def test_dx_repeated_solves(tca):
    """The P ping-pong restarts at every solve; cached graphs stay valid."""
    n, m, lam = (32, 32, 32, 15), (64, 64, 64, 30), 1e-2
    A, L = synth.mode_matrices(n, m, seed=2)
    o = oracle.Operator(A, L, lam)
    op = tca.Operator(A, L, lam, dtype="f32")
    for seed, k in ((3, 33), (4, 64), (5, 7), (6, 40)):
        b = synth.random_tensor(n, seed=seed)
        os.environ.update(GENERAL)
        try:
            xg, rep = op.cg_solve(dev(b, "f32"), rtol=0.0, max_iters=k)
        finally:
            for kk in GENERAL:
                os.environ.pop(kk, None)
        assert op.cg_deferred_x is True   # the fp32 default
        xr, _, _, _ = o.cg(b, rtol=0.0, max_iters=k)
        assert rep["iterations"] == k
        assert rel(xg.double().cpu().numpy(), xr) <= 2e-5
    op.close()
