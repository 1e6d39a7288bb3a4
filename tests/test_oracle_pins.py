"""Pins of the CPU oracle to things other than itself (P1-P9).

Every check here compares oracle/ against the paper's printed values, closed
forms, textbook spectra, brute-force assembly or numpy's independent dense
linear algebra -- never against the oracle re-typed.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
import synth
from conftest import read_golden

TINY_SHAPES = [((5, 4, 3), (8, 7, 6)), ((4, 3, 3, 2), (6, 5, 5, 4)), ((7,), (11,)),
               ((6, 5), (9, 9))]


def brute_force_K(A, L, lam):
    """Assemble K = kron_d G_d + lam sum_d (I..R_d..I) entry by entry with
    index loops (G_d, R_d from numpy matmul, independent of the oracle)."""
    D = len(A)
    n = [a.shape[1] for a in A]
    G = [a.T @ a for a in A]
    R = [(l.T @ l) if l is not None and l.shape[0] else np.zeros((nd, nd)) for l, nd in zip(L, n)]
    N = int(np.prod(n))
    K = np.zeros((N, N))
    idx = list(itertools.product(*[range(nd) for nd in n]))
    for I, i in enumerate(idx):
        for J, j in enumerate(idx):
            v = 1.0
            for d in range(D):
                v *= G[d][i[d], j[d]]
            reg = 0.0
            for d in range(D):
                if all(i[e] == j[e] for e in range(D) if e != d):
                    reg += R[d][i[d], j[d]]
            K[I, J] = v + lam * reg
    return K


def tiny_problem(n, m, seed=3, lam=0.05, basis="bspline"):
    A, L = synth.mode_matrices(n, m, basis=basis, seed=seed)
    return A, L, oracle.Operator(A, L, lam)


# ---------------------------------------------------------------- P1
@pytest.mark.parametrize("n,m", TINY_SHAPES)
@pytest.mark.parametrize("basis", ["bspline", "gauss"])
def test_P1_apply_equals_bruteforce_kronecker(n, m, basis):
    A, L, op = tiny_problem(n, m, basis=basis)
    K = brute_force_K(A, L, op.lam)
    x = synth.random_tensor(n, seed=11)
    y = op.apply(x)
    ref = K @ x.ravel()
    assert np.linalg.norm(y.ravel() - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("n,m", TINY_SHAPES[:2])
def test_P1_cg_equals_dense_direct_solve(n, m):
    A, L, op = tiny_problem(n, m)
    K = brute_force_K(A, L, op.lam)
    b = synth.random_tensor(n, seed=12)
    x, it, st, hist = op.cg(b, rtol=1e-14, max_iters=2000)
    assert st == oracle.OK
    xd = np.linalg.solve(K, b.ravel())
    assert np.linalg.norm(x.ravel() - xd) <= 1e-10 * np.linalg.norm(xd)
    assert len(hist) == it + 1


def test_P1_mode_product_against_einsum_nonsymmetric():
    rng = np.random.default_rng(5)
    X = rng.standard_normal((3, 4, 5, 2))
    for d in range(4):
        M = rng.standard_normal((7, X.shape[d]))  # rectangular, not symmetric
        Y = oracle.mode_product(X, d, M)
        sub = "abcd"
        out = sub.replace(sub[d], "z")
        ref = np.einsum(f"z{sub[d]},{sub}->{out}", M, X)
        assert np.allclose(Y, ref, rtol=1e-14, atol=1e-14)


def test_P1_apply_point_matches_apply():
    n, m = (6, 5, 7, 4), (12, 10, 13, 8)
    A, L, op = tiny_problem(n, m, lam=0.3)
    x = synth.random_tensor(n, seed=13)
    y = op.apply(x)
    for i in [(0, 0, 0, 0), (5, 4, 6, 3), (2, 1, 3, 2), (0, 4, 1, 3), (5, 0, 6, 0)]:
        assert abs(op.apply_point(x, i) - y[i]) <= 1e-13 * np.abs(y).max()


def test_P1_gram_by_loops_equals_matmul():
    A = synth.gaussian_matrix(9, 13, seed=2, mode=0)
    assert np.allclose(oracle.gram(A), A.T @ A, rtol=1e-14, atol=1e-15)


def test_dot_against_exactly_rounded_sum():
    a = synth.random_tensor((10001,), seed=1)
    b = synth.random_tensor((10001,), seed=2, stream=8)
    exact = math.fsum(a * b)  # products rounded, then exact sum
    assert abs(oracle.dot(a, b) - exact) <= 1e-13 * math.fsum(np.abs(a * b))
    assert oracle.dot(a[:0], b[:0]) == 0.0


# ---------------------------------------------------------------- P2
@pytest.mark.parametrize("cfg", [0, 2])
def test_P2_symmetry_normwise_and_positive(cfg):
    c = synth.CONFIGS[cfg]
    A, L = synth.mode_matrices(c)
    op = oracle.Operator(A, L, c.lam)
    x = synth.random_tensor(c.n, seed=21)
    y = synth.random_tensor(c.n, seed=22, stream=8)
    Mx, My = op.apply(x), op.apply(y)
    a = oracle.dot(x, My)
    b = oracle.dot(Mx, y)
    assert abs(a - b) <= 1e-13 * np.linalg.norm(x) * np.linalg.norm(My)
    assert oracle.dot(x, Mx) > 0


def test_P2_tiny_K_from_oracle_columns_symmetric_pd():
    n, m = (4, 3, 3), (6, 5, 5)
    A, L, op = tiny_problem(n, m, lam=0.1)
    N = op.N
    K = np.empty((N, N))
    for j in range(N):
        e = np.zeros(N)
        e[j] = 1.0
        K[:, j] = op.apply(e.reshape(n)).ravel()
    assert np.abs(K - K.T).max() <= 1e-15 * np.abs(K).max()
    assert np.linalg.eigvalsh(K).min() > 0


# ---------------------------------------------------------------- P3
def test_P3_recovery_noiseless_unregularised():
    c = synth.CONFIGS[0]
    A, L = synth.mode_matrices(c)
    op = oracle.Operator(A, None, 0.0)
    xt = synth.x_true(c.n, seed=1)
    y = synth.forward_model(A, xt)
    b = op.rhs(y)
    x, it, st, _ = op.cg(b, rtol=1e-14, max_iters=5000)
    assert st == oracle.OK
    assert np.linalg.norm(x - xt) <= 1e-9 * np.linalg.norm(xt)


# ---------------------------------------------------------------- P4
def test_P4_separability_eigenvectors_of_G():
    n, m = (5, 4, 6, 3), (9, 8, 11, 7)
    A, _ = synth.mode_matrices(n, m)
    op = oracle.Operator(A, None, 0.0)
    G = [a.T @ a for a in A]
    rng = np.random.default_rng(0)
    for _ in range(3):
        vs, mus = [], []
        for Gd in G:
            w, V = np.linalg.eigh(Gd)
            k = rng.integers(len(w))
            vs.append(V[:, k])
            mus.append(w[k])
        x = vs[0]
        for v in vs[1:]:
            x = np.multiply.outer(x, v)
        y = op.apply(x)
        assert np.allclose(y, np.prod(mus) * x, atol=1e-13 * np.abs(np.prod(mus)))


def test_P4_kronecker_sum_spectrum_of_regulariser():
    n = (6, 5, 7)
    A = [np.eye(nd) for nd in n]  # G_d = I
    L = [synth.second_difference(nd) for nd in n]
    lam = 0.7
    op = oracle.Operator(A, L, lam)
    vs, nus = [], []
    for l in L:
        w, V = np.linalg.eigh(l.T @ l)
        vs.append(V[:, -1])
        nus.append(w[-1])
    x = np.multiply.outer(np.multiply.outer(vs[0], vs[1]), vs[2])
    y = op.apply(x)
    assert np.allclose(y, (1.0 + lam * sum(nus)) * x, atol=1e-13 * (1 + lam * sum(nus)))


def test_P4_rank1_separable_transformation():
    """Eq. 4: a separable operator maps a rank-1 tensor to the rank-1 tensor of
    the per-mode images."""
    n, m = (5, 4, 3), (8, 7, 6)
    A, _ = synth.mode_matrices(n, m, basis="gauss", seed=4)
    op = oracle.Operator(A, None, 0.0)
    G = [a.T @ a for a in A]
    rng = np.random.default_rng(1)
    v = [rng.standard_normal(nd) for nd in n]
    x = np.multiply.outer(np.multiply.outer(v[0], v[1]), v[2])
    gv = [G[d] @ v[d] for d in range(3)]
    ref = np.multiply.outer(np.multiply.outer(gv[0], gv[1]), gv[2])
    assert np.allclose(op.apply(x), ref, rtol=1e-13, atol=1e-14)


# ---------------------------------------------------------------- P5
def test_P5_commutativity_all_mode_orders():
    n = (5, 4, 6, 3)
    rng = np.random.default_rng(2)
    X = rng.standard_normal(n)
    mats = [rng.standard_normal((nd, nd)) for nd in n]  # not symmetric
    results = []
    for perm in itertools.permutations(range(4)):
        Y = X
        for d in perm:
            Y = oracle.mode_product(Y, d, mats[d])
        results.append(Y)
    ref = results[0]
    for Y in results[1:]:
        assert np.linalg.norm(Y - ref) <= 1e-13 * np.linalg.norm(ref)


# ---------------------------------------------------------------- P6
def test_P6_second_difference_gram_closed_form():
    g = read_golden("second_difference_gram.txt")
    n = int(g["n"])
    R = oracle.gram(synth.second_difference(n))
    for key in ("row0", "row1", "row3", "row6"):
        want = np.array([float(v) for v in g[key].split()])
        assert np.array_equal(R[int(key[3:])], want)
    assert np.abs(R @ np.ones(n)).max() == 0.0
    assert np.abs(R @ np.arange(n, dtype=float)).max() == 0.0


def test_P6_bspline_closed_form_values():
    g = read_golden("bspline_values.txt")
    u = np.array([float(v) for v in g["u"].split()])
    want = np.array([float(v) for v in g["beta3"].split()])
    assert np.allclose(synth.cubic_bspline(u), want, rtol=0, atol=1e-16)


def _cox_de_boor(t, knots, i, k):
    if k == 0:
        return 1.0 if knots[i] <= t < knots[i + 1] else 0.0
    a = (t - knots[i]) / (knots[i + k] - knots[i])
    b = (knots[i + k + 1] - t) / (knots[i + k + 1] - knots[i + 1])
    return a * _cox_de_boor(t, knots, i, k - 1) + b * _cox_de_boor(t, knots, i + 1, k - 1)


@pytest.mark.parametrize("n,m", [(12, 20), (16, 32), (15, 30)])
def test_P6_bspline_matrix_vs_cox_de_boor_and_partition(n, m):
    A = synth.bspline_matrix(n, m)
    t = synth.sample_positions(n, m)
    for i in range(m):
        for k in range(n):
            knots = [k - 2, k - 1, k, k + 1, k + 2]
            assert abs(A[i, k] - _cox_de_boor(t[i], knots, 0, 3)) <= 1e-15
    inner = (t >= 1) & (t <= n - 2)
    assert np.allclose(A[inner].sum(axis=1), 1.0, atol=1e-15)
    assert np.count_nonzero(A, axis=1).max() <= 4


# ---------------------------------------------------------------- P7
def test_P7_paper_printed_band_count():
    g = read_golden("paper_band_count.txt")
    grid = [int(v) for v in g["grid"].split()]
    total = 1
    for nd in grid:
        G = oracle.gram(synth.bspline_matrix(nd, 2 * nd))
        upper = int(np.count_nonzero(np.triu(G)))
        assert upper == 4 * nd - 6
        total *= upper
    assert total == int(g["nonzeros"])
    assert round(total * 4 / 1e9) == int(g["gbytes_single"])


# ---------------------------------------------------------------- P8
def test_P8_rhs_of_forward_model_equals_unregularised_apply():
    n, m = (6, 5, 4, 3), (12, 10, 8, 6)
    A, _ = synth.mode_matrices(n, m)
    op = oracle.Operator(A, None, 0.0)
    x = synth.random_tensor(n, seed=31)
    lhs = op.rhs(synth.forward_model(A, x))
    rhs = op.apply(x)
    assert np.linalg.norm(lhs - rhs) <= 1e-13 * np.linalg.norm(rhs)


def test_P8_rank1_rhs_and_pointwise():
    n, m = (5, 4, 3), (8, 7, 6)
    A, _ = synth.mode_matrices(n, m, basis="gauss", seed=9)
    op = oracle.Operator(A, None, 0.0)
    rng = np.random.default_rng(3)
    u = [rng.standard_normal(md) for md in m]
    y = np.multiply.outer(np.multiply.outer(u[0], u[1]), u[2])
    b = op.rhs(y)
    au = [A[d].T @ u[d] for d in range(3)]
    ref = np.multiply.outer(np.multiply.outer(au[0], au[1]), au[2])
    assert np.allclose(b, ref, rtol=1e-13, atol=1e-14)
    for i in [(0, 0, 0), (4, 3, 2), (2, 1, 1)]:
        assert abs(op.rhs_point(y, i) - b[i]) <= 1e-13 * np.abs(b).max()


# ---------------------------------------------------------------- P9
def test_P9_spec_worked_example_cg():
    g = read_golden("spec_cg_example.txt")
    T = np.array([[float(v) for v in row.split()] for row in g["matrix"].split(";")])
    A1 = np.linalg.cholesky(T).T  # upper factor: A1^T A1 = T
    ones = np.array([float(v) for v in g["b"].split()])
    y = np.linalg.solve(A1.T, ones)  # A1^T y = 1
    op = oracle.Operator([A1], None, 0.0)
    b = op.rhs(y)
    assert np.allclose(b, ones, atol=1e-14)
    x, it, st, hist = op.cg(b, rtol=1e-15, max_iters=int(g["max_iters"]))
    want = np.array([float(v) for v in g["x"].split()])
    assert st == oracle.OK
    assert np.abs(x - want).max() <= 1e-12
    assert it <= int(g["max_iters"])


def test_cg_zero_rhs_zero_iterations():
    A, L, op = tiny_problem((4, 3, 3), (6, 5, 5))
    x, it, st, hist = op.cg(np.zeros(op.n), rtol=1e-10, max_iters=10)
    assert it == 0 and st == oracle.OK and np.all(x == 0)


def test_cg_rho_zero_guard_and_history_decrease():
    # order-1 diagonal system: CG converges exactly in 1 step, rho == 0 (Z12 guard)
    op = oracle.Operator([np.diag([2.0, 2.0, 2.0])], None, 0.0)
    x, it, st, hist = op.cg(np.ones(3), rtol=0.0, max_iters=5)
    assert st == oracle.OK and it == 1 and hist[-1] == 0.0
    assert np.allclose(x, 0.25)
    c = synth.CONFIGS[0]
    A, L = synth.mode_matrices(c)
    op = oracle.Operator(A, L, c.lam)
    b = op.rhs(synth.data(A, c.n, c.m))
    x, it, st, hist = op.cg(b, rtol=c.rtol, max_iters=c.max_iters)
    assert st == oracle.OK and hist[-1] <= c.rtol ** 2 * hist[0]
    assert np.all(hist[1:] <= 10 * np.maximum.accumulate(hist)[:-1])
    r = b - op.apply(x)
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(b)


def test_cg_not_converged_status():
    c = synth.CONFIGS[0]
    A, L = synth.mode_matrices(c)
    op = oracle.Operator(A, L, c.lam)
    b = op.rhs(synth.data(A, c.n, c.m))
    x, it, st, hist = op.cg(b, rtol=1e-30, max_iters=5)
    assert st == oracle.NOT_CONVERGED and it == 5


def test_thread_count_independent():
    import os
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import numpy as np, oracle, synth;"
            "c=synth.CONFIGS[2]; A,L=synth.mode_matrices(c); op=oracle.Operator(A,L,c.lam);"
            "x=synth.random_tensor(c.n,5); y=op.apply(x); print(repr(oracle.dot(y,y)))"
            % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    outs = []
    for t in ("1", "3"):
        env = dict(os.environ, OMP_NUM_THREADS=t)
        outs.append(subprocess.check_output([sys.executable, "-c", code], env=env).strip())
    assert outs[0] == outs[1]


# ---------------------------------------------------------------- P10-P13: Kronecker-factor PCG (reading Z22)
def dense_precond(op):
    """P = kron_d F_d with F_d = G_d + eps_d R_d formed with numpy (eigvalsh for
    gbar, matmul Grams): independent of the oracle's Cholesky-based route."""
    G = [a.T @ a for a in op.A]
    gbar = [float(np.exp(np.mean(np.log(np.linalg.eigvalsh(g))))) for g in G]
    F = []
    for d in range(op.D):
        eps = op.lam / float(np.prod([gbar[e] for e in range(op.D) if e != d]))
        R = op.R[d] if op.R[d] is not None else np.zeros_like(G[d])
        F.append(G[d] + eps * R)
    P = np.ones((1, 1))
    for f in F:
        P = np.kron(P, f)
    return F, P


@pytest.mark.parametrize("n,m", TINY_SHAPES)
def test_P10_geomean_eigenvalue_against_eigvalsh(n, m):
    A, L, op = tiny_problem(n, m)
    for g in op.G:
        ref = float(np.exp(np.mean(np.log(np.linalg.eigvalsh(g)))))
        assert abs(oracle.geomean_eig(g) - ref) <= 1e-13 * ref
    F, eps = op.precond_factors()
    Fr, _ = dense_precond(op)
    for f, fr in zip(F, Fr):
        assert np.abs(f - fr).max() <= 1e-13 * np.abs(fr).max()


@pytest.mark.parametrize("n,m", TINY_SHAPES)
@pytest.mark.parametrize("basis", ["bspline", "gauss"])
def test_P11_precond_apply_equals_dense_kronecker_solve(n, m, basis):
    A, L, op = tiny_problem(n, m, basis=basis)
    F, P = dense_precond(op)
    r = synth.random_tensor(n, seed=13)
    z = op.precond_apply(r)
    # the dense Kronecker solve carries kappa(P) = prod kappa(F_d) rounding
    ref = np.linalg.solve(P, r.ravel())
    tol = max(1e-12, 1e-15 * np.linalg.cond(P))
    assert np.linalg.norm(z.ravel() - ref) <= tol * np.linalg.norm(ref)
    # one-dimensional numpy solves along each mode (Eq. 4 order)
    zz = r.copy()
    for d, f in enumerate(F):
        t = np.moveaxis(zz, d, 0)
        zz = np.moveaxis(np.linalg.solve(f, t.reshape(f.shape[0], -1)).reshape(t.shape), 0, d)
    tol1 = max(1e-12, 1e-14 * sum(np.linalg.cond(f) for f in F))   # per-solve rounding x kappa(F_d)
    assert np.linalg.norm(z - zz) <= tol1 * np.linalg.norm(zz)
    # P^-1 is symmetric: <s, P^-1 r> = <P^-1 s, r>
    s = synth.random_tensor(n, seed=14)
    a, b = oracle.dot(s, z), oracle.dot(op.precond_apply(s), r)
    assert abs(a - b) <= 1e-13 * np.linalg.norm(s) * np.linalg.norm(z)


@pytest.mark.parametrize("n,m,lam", [((9,), (15,), 0.05), ((5, 4, 3), (8, 7, 6), 0.0),
                                     ((4, 3, 3, 2), (6, 5, 5, 4), 0.0)])
def test_P12_exact_preconditioner_converges_in_one_iteration(n, m, lam):
    """D = 1: F_1 = G_1 + lam R_1 = M (empty product, eps = lam); lam = 0:
    P = kron G_d = M.  Either way P = M and PCG stops after one step at M^-1 b."""
    A, L, op = tiny_problem(n, m, lam=lam)
    K = brute_force_K(A, L, lam)
    b = synth.random_tensor(n, seed=17)
    x, k, st, hist = op.pcg(b, rtol=1e-12, max_iters=10)
    assert st == oracle.OK and k == 1
    ref = np.linalg.solve(K, b.ravel())
    assert np.linalg.norm(x.ravel() - ref) <= 1e-12 * np.linalg.norm(ref)


# (the tiny 4-D Gaussian case is left out: its gbar_e ~ 0.03 make eps_d ~ 500, so
# F_d ~ eps_d R_d is near-singular (kappa(P) ~ 1e16) and PCG stagnates -- a
# property of the preconditioner (Z22), not of the iteration)
@pytest.mark.parametrize("n,m,basis", [((5, 4, 3), (8, 7, 6), "bspline"), ((5, 4, 3), (8, 7, 6), "gauss"),
                                       ((4, 3, 3, 2), (6, 5, 5, 4), "bspline"), ((6, 5), (9, 9), "bspline"),
                                       ((6, 5), (9, 9), "gauss")])
def test_P13_pcg_equals_dense_direct_solve(n, m, basis):
    A, L, op = tiny_problem(n, m, basis=basis)
    K = brute_force_K(A, L, op.lam)
    b = synth.random_tensor(n, seed=19)
    x, k, st, hist = op.pcg(b, rtol=1e-14, max_iters=500)
    ref = np.linalg.solve(K, b.ravel())
    assert st == oracle.OK
    tol = max(1e-10, 1e-14 * np.linalg.cond(K))
    assert np.linalg.norm(x.ravel() - ref) <= tol * np.linalg.norm(ref)
    assert hist[-1] <= 1e-28 * hist[0]


def test_P13_pcg_fewer_iterations_than_cg_on_config0():
    cfg = synth.CONFIGS[0]
    A, L = synth.mode_matrices(cfg)
    op = oracle.Operator(A, L, cfg.lam)
    b = op.rhs(synth.data(A, cfg.n, cfg.m, seed=1))
    _, kc, stc, _ = op.cg(b, rtol=cfg.rtol, max_iters=cfg.max_iters)
    x, kp, stp, hist = op.pcg(b, rtol=cfg.rtol, max_iters=cfg.max_iters)
    assert stc == stp == oracle.OK
    assert kp < kc
    assert hist[-1] <= cfg.rtol ** 2 * hist[0]


# ---------------------------------------------------------------- P14: single-reduction CG (reading Z24)
@pytest.mark.parametrize("n,m", TINY_SHAPES[:2] + [((6, 5), (9, 9))])
@pytest.mark.parametrize("basis", ["bspline", "gauss"])
def test_P14_cgsr_equals_dense_direct_solve(n, m, basis):
    A, L, op = tiny_problem(n, m, basis=basis)
    K = brute_force_K(A, L, op.lam)
    b = synth.random_tensor(n, seed=23)
    x, k, st, hist = op.cgsr(b, rtol=1e-14, max_iters=3000)
    ref = np.linalg.solve(K, b.ravel())
    assert st == oracle.OK
    tol = max(1e-10, 1e-14 * np.linalg.cond(K))
    assert np.linalg.norm(x.ravel() - ref) <= tol * np.linalg.norm(ref)


def test_P14_cgsr_spec_worked_example():
    """SPEC.md:495 example through the single-reduction recurrences: exact at
    k = 2 with gamma = 0 (the Z12 guard)."""
    g = read_golden("spec_cg_example.txt")
    T = np.array([[float(v) for v in row.split()] for row in g["matrix"].split(";")])
    A1 = np.linalg.cholesky(T).T
    ones = np.array([float(v) for v in g["b"].split()])
    op = oracle.Operator([A1], None, 0.0)
    b = op.rhs(np.linalg.solve(A1.T, ones))
    x, it, st, hist = op.cgsr(b, rtol=1e-15, max_iters=int(g["max_iters"]))
    want = np.array([float(v) for v in g["x"].split()])
    assert st == oracle.OK and it <= int(g["max_iters"])
    assert np.abs(x - want).max() <= 1e-12


@pytest.mark.parametrize("cfg_index", [0, 2])
def test_P14_cgsr_iterates_match_fig2_cg_to_rounding(cfg_index):
    """Same Krylov iterates as Fig. 2 in exact arithmetic: at matched k the two
    recurrences differ only by rounding on these well-conditioned systems."""
    cfg = synth.CONFIGS[cfg_index]
    A, L = synth.mode_matrices(cfg)
    op = oracle.Operator(A, L, cfg.lam)
    b = op.rhs(synth.data(A, cfg.n, cfg.m, seed=1))
    for k in (5, 30):
        xa, _, _, ha = op.cg(b, rtol=0.0, max_iters=k)
        xb, _, _, hb = op.cgsr(b, rtol=0.0, max_iters=k)
        assert np.linalg.norm(xa - xb) <= 1e-10 * np.linalg.norm(xa)
        assert np.max(np.abs(ha - hb) / ha) <= 1e-9


# ---------------------------------------------------------------- P15: separable Poisson + tensor Jacobi (Z25, Z26)
def dense_poisson(n):
    """sum_d I..T_d..I with numpy kron (independent of the oracle)."""
    T = [synth.laplacian_1d(k) for k in n]
    K = 0
    for d in range(len(n)):
        P = np.ones((1, 1))
        for e in range(len(n)):
            P = np.kron(P, T[e] if e == d else np.eye(n[e]))
        K = K + P
    return K


@pytest.mark.parametrize("n", [(5, 6, 7), (4, 3, 5, 2), (9,)])
def test_P15_poisson_apply_equals_dense_kronecker_sum(n):
    o = oracle.Operator.from_gram(None, [synth.laplacian_1d(k) for k in n], 1.0)
    x = synth.random_tensor(n, seed=31)
    ref = dense_poisson(n) @ x.ravel()
    assert np.linalg.norm(o.apply(x).ravel() - ref) <= 1e-14 * np.linalg.norm(ref)


def test_P15_poisson_textbook_spectrum():
    """Eigen-tensors of the Dirichlet Laplacian: prod_d sin(k_d pi (i_d+1)/(n_d+1))
    with eigenvalue sum_d (2 - 2 cos(k_d pi / (n_d+1)))."""
    n = (7, 6, 9)
    o = oracle.Operator.from_gram(None, [synth.laplacian_1d(k) for k in n], 1.0)
    for ks in [(1, 1, 1), (3, 5, 2), (7, 6, 9)]:
        vs = [np.sin(k * np.pi * (np.arange(nd) + 1) / (nd + 1)) for k, nd in zip(ks, n)]
        lam = sum(2 - 2 * np.cos(k * np.pi / (nd + 1)) for k, nd in zip(ks, n))
        x = np.multiply.outer(np.multiply.outer(vs[0], vs[1]), vs[2])
        assert np.allclose(o.apply(x), lam * x, atol=1e-13 * lam)


@pytest.mark.parametrize("n", [(5, 6, 7), (4, 3, 5, 2)])
def test_P15_jacobi_steps_and_solution(n):
    """Fig. 1: U_{k+1} = U_k - (K U_k - b) / diag(K) (numpy, first steps) and the
    converged U equals the dense solve; the residual history is R+*R."""
    K = dense_poisson(n)
    o = oracle.Operator.from_gram(None, [synth.laplacian_1d(k) for k in n], 1.0)
    b = synth.random_tensor(n, seed=32).ravel()
    u = np.zeros_like(b)
    hist = []
    for _ in range(3):
        r = K @ u - b
        hist.append(r @ r)
        u = u - r / np.diag(K)
    uo, k, st, h = o.jacobi(b.reshape(n), threshold=0.0, max_iters=3)
    assert st == oracle.NOT_CONVERGED and k == 3
    assert np.linalg.norm(uo.ravel() - u) <= 1e-14 * np.linalg.norm(u)
    assert np.allclose(h[:3], hist, rtol=1e-13)
    uo, k, st, h = o.jacobi(b.reshape(n), threshold=1e-24, max_iters=50000)
    ref = np.linalg.solve(K, b)
    assert st == oracle.OK and h[-1] <= 1e-24
    assert np.linalg.norm(uo.ravel() - ref) <= 1e-9 * np.linalg.norm(ref)


# ---------------------------------------------------------------- P16: scattered-data operator (reading Z27)
def scipy_sample_matrix(n, t):
    """Dense K x N sample matrix W[k, i] = prod_d beta3(t[k,d] - i_d), the cubic
    B-spline from scipy's BSpline.basis_element on knots (-2,-1,0,1,2) (an
    evaluation independent of the oracle's)."""
    from scipy.interpolate import BSpline
    b = BSpline.basis_element([-2.0, -1.0, 0.0, 1.0, 2.0], extrapolate=False)
    per = []
    for d, nd in enumerate(n):
        v = b(t[:, d][:, None] - np.arange(nd)[None, :])
        per.append(np.nan_to_num(v, nan=0.0))
    W = per[0]
    for d in range(1, len(n)):
        W = (W[:, :, None] * per[d][:, None, :]).reshape(t.shape[0], -1)
    return W


@pytest.mark.parametrize("n,K", [((5, 4, 6), 40), ((4, 3, 5, 6), 60), ((9,), 7), ((6, 7), 25)])
def test_P16_scattered_equals_dense_sample_matrix(n, K):
    t = synth.scattered_positions(n, K, seed=3)
    t[0] = np.floor(t[0])   # a sample on grid points (3 nonzeros per mode)
    W = scipy_sample_matrix(n, t)
    L = [synth.second_difference(k) for k in n]
    o = oracle.ScatteredOperator(n, t, L, 0.1)
    x = synth.random_tensor(n, seed=41).ravel()
    yk = synth.random_tensor((K,), seed=42)
    R = 0
    for d in range(len(n)):
        P = np.ones((1, 1))
        for e in range(len(n)):
            P = np.kron(P, (L[e].T @ L[e]) if e == d else np.eye(n[e]))
        R = R + P
    ref = W.T @ (W @ x) + 0.1 * (R @ x)
    assert np.linalg.norm(o.apply(x).ravel() - ref) <= 1e-14 * np.linalg.norm(ref)
    assert np.linalg.norm(o.rhs(yk).ravel() - W.T @ yk) <= 1e-14 * np.linalg.norm(W.T @ yk)
    assert np.linalg.norm(o.forward(x) - W @ x) <= 1e-14 * np.linalg.norm(W @ x)


def test_P16_full_grid_samples_equal_kronecker_operator():
    """Samples on the whole tensor grid of Z5's positions: sum_k w_k w_k^T =
    kron_d A_d^T A_d and sum_k y_k w_k = (kron A_d^T) y (Eq. 4), the gridded
    operator pinned by P1-P7."""
    n, m = (6, 5, 7), (11, 9, 12)
    A, L = synth.mode_matrices(n, m)
    pos = [synth.sample_positions(nd, md) for nd, md in zip(n, m)]
    t = np.array(list(itertools.product(*pos)))
    so = oracle.ScatteredOperator(n, t, L, 1e-2)
    go = oracle.Operator(A, L, 1e-2)
    x = synth.random_tensor(n, seed=43)
    ref = go.apply(x)
    assert np.linalg.norm(so.apply(x) - ref) <= 1e-13 * np.linalg.norm(ref)
    y = synth.random_tensor(m, seed=44)
    ref = go.rhs(y)
    assert np.linalg.norm(so.rhs(y.ravel()) - ref) <= 1e-13 * np.linalg.norm(ref)


def test_P16_partition_of_unity_and_energy():
    """sum_i beta3(t - i) = 1 for t in [1, n-2] (cubic B-spline partition of
    unity): W 1 = 1 on interior samples; <x, W^T W x> = ||W x||^2 >= 0."""
    n = (8, 9, 7, 6)
    t = synth.scattered_positions(n, 300, seed=5)
    o = oracle.ScatteredOperator(n, t, None, 0.0)
    one = o.forward(np.ones(n))
    inside = np.all((t >= 1.0) & (t <= np.asarray(n) - 2.0), axis=1)
    assert inside.sum() > 20
    assert np.allclose(one[inside], 1.0, rtol=0, atol=1e-14)
    assert np.all(one[~inside] < 1.0 + 1e-14)
    x = synth.random_tensor(n, seed=45)
    wx = o.forward(x)
    assert np.isclose(float(np.sum(x * o.data(x))), float(wx @ wx), rtol=1e-13)


def test_P16_scattered_cg_equals_dense_solve():
    n = (5, 4, 6, 3)
    t = synth.scattered_positions(n, 500, seed=6)
    L = [synth.second_difference(k) for k in n]
    o = oracle.ScatteredOperator(n, t, L, 1e-2)
    W = scipy_sample_matrix(n, t)
    R = 0
    for d in range(len(n)):
        P = np.ones((1, 1))
        for e in range(len(n)):
            P = np.kron(P, (L[e].T @ L[e]) if e == d else np.eye(n[e]))
        R = R + P
    M = W.T @ W + 1e-2 * R
    b = synth.random_tensor(n, seed=46)
    x, k, st, hist = o.cg(b, rtol=1e-13, max_iters=2000)
    assert st == oracle.OK
    ref = np.linalg.solve(M, b.ravel())
    assert np.linalg.norm(x.ravel() - ref) <= 1e-9 * np.linalg.norm(ref)


# ---------------------------------------------------------------- P17: warm start (Fig. 2's R := B - A*C with C != 0)
def _numpy_cg(K, b, x0, k):
    """Textbook CG (the recurrences of Fig. 2) in numpy on a
    dense SPD matrix, k steps from x0."""
    x = x0.copy()
    r = b - K @ x
    p = r.copy()
    rho = r @ r
    for _ in range(k):
        q = K @ p
        alpha = rho / (p @ q)
        x = x + alpha * p
        r = r - alpha * q
        rho1 = r @ r
        p = r + (rho1 / rho) * p
        rho = rho1
    return x


@pytest.mark.parametrize("n,m", TINY_SHAPES)
def test_P17_warm_start_iterates_equal_dense_cg_and_first_step_is_steepest_descent(n, m):
    """R := B - A*C, P := R.  Step 1 from C is the exact
    steepest-descent step x1 = x0 + (r0.r0 / r0.K r0) r0 (closed form), and
    steps 2..4 equal textbook CG on the brute-force K from the same x0."""
    A, L, op = tiny_problem(n, m)
    K = brute_force_K(A, L, op.lam)
    b = synth.random_tensor(n, seed=31)
    x0 = synth.random_tensor(n, seed=32, stream=8)
    r0 = b.ravel() - K @ x0.ravel()
    x1_ref = x0.ravel() + (r0 @ r0) / (r0 @ K @ r0) * r0
    x1, k1, st, hist = op.cg(b, rtol=0.0, max_iters=1, x0=x0)
    assert k1 == 1 and st == oracle.OK
    assert abs(hist[0] - r0 @ r0) <= 1e-12 * (r0 @ r0)          # rho_0 = <B - A C, B - A C>
    assert np.linalg.norm(x1.ravel() - x1_ref) <= 1e-12 * np.linalg.norm(x1_ref)
    for k in (2, 3, 4):
        xk, _, _, _ = op.cg(b, rtol=0.0, max_iters=k, x0=x0)
        ref = _numpy_cg(K, b.ravel(), x0.ravel(), k)
        assert np.linalg.norm(xk.ravel() - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("solver", ["cg", "pcg", "cgsr"])
def test_P17_warm_start_converges_to_dense_solve_with_b_relative_stop(solver):
    """Warm start to tolerance: the stop reference is <b, b> (reading Z28), and
    the converged solution is the dense direct solve of the brute-force K."""
    n, m = (5, 4, 3), (8, 7, 6)
    A, L, op = tiny_problem(n, m)
    K = brute_force_K(A, L, op.lam)
    b = synth.random_tensor(n, seed=33)
    x0 = 3.0 * synth.random_tensor(n, seed=34, stream=8)
    x, k, st, hist = getattr(op, solver)(b, rtol=1e-12, max_iters=2000, x0=x0)
    assert st == oracle.OK
    assert hist[-1] <= 1e-24 * float(b.ravel() @ b.ravel())
    ref = np.linalg.solve(K, b.ravel())
    assert np.linalg.norm(x.ravel() - ref) <= 1e-9 * np.linalg.norm(ref)
    # started at the solution: the initial residual is rounding-level and one step ends it
    xs, ks, sts, hs = getattr(op, solver)(b, rtol=1e-8, max_iters=50, x0=ref.reshape(n))
    assert sts == oracle.OK and ks <= 1
    assert np.linalg.norm(xs.ravel() - ref) <= 1e-12 * np.linalg.norm(ref)


# ---------------------------------------------------------------- P18: PCG iterates (reading Z22)
@pytest.mark.parametrize("n,m", TINY_SHAPES[:2] + [((6, 5), (9, 9))])
def test_P18_pcg_iterates_equal_cg_on_split_preconditioned_system(n, m):
    """Preconditioned CG with P = C C^T produces x_k = C^-T xh_k where xh_k are
    plain CG iterates on (C^-1 K C^-T) xh = C^-1 b (textbook equivalence).  P =
    kron F_d, F_d = G_d + eps_d R_d with G_d, R_d, gbar from numpy only (reading
    Z22).  A beta built from <r, r> instead of <r, z> fails this from k = 2 on."""
    A, L, op = tiny_problem(n, m)
    K = brute_force_K(A, L, op.lam)
    G = [a.T @ a for a in A]
    R = [l.T @ l if l is not None and l.shape[0] else np.zeros_like(g) for l, g in zip(L, G)]
    gbar = [float(np.exp(np.mean(np.log(np.linalg.eigvalsh(g))))) for g in G]
    P = np.ones((1, 1))
    for d in range(len(G)):
        eps = op.lam / float(np.prod([gbar[e] for e in range(len(G)) if e != d]))
        P = np.kron(P, G[d] + eps * R[d])
    C = np.linalg.cholesky(P)
    Ci = np.linalg.inv(C)
    Kh = Ci @ K @ Ci.T
    b = synth.random_tensor(n, seed=35).ravel()
    bh = Ci @ b

    def wrong_beta_pcg(k):   # beta = <r1, r1> / <r, r> with z = P^-1 r directions
        x = np.zeros_like(b)
        r = b.copy()
        z = np.linalg.solve(P, r)
        p = z.copy()
        rho, rr = r @ z, r @ r
        for _ in range(k):
            q = K @ p
            alpha = rho / (p @ q)
            x, r = x + alpha * p, r - alpha * q
            z = np.linalg.solve(P, r)
            rr1 = r @ r
            p = z + (rr1 / rr) * p
            rho, rr = r @ z, rr1
        return x

    for k in (1, 2, 3, 4):
        xk, kk, st, _ = op.pcg(b.reshape(n), rtol=0.0, max_iters=k)
        assert kk == k and st == oracle.OK
        ref = Ci.T @ _numpy_cg(Kh, bh, np.zeros_like(bh), k)
        err = np.linalg.norm(xk.ravel() - ref) / np.linalg.norm(ref)
        assert err <= 1e-10
        if k >= 2:   # the pin discriminates the preconditioned beta
            wrong = wrong_beta_pcg(k)
            assert np.linalg.norm(wrong - ref) / np.linalg.norm(ref) > 1e3 * max(err, 1e-14)
