"""Scattered-data operator (reading Z27): the GPU sample-term
kernels through the C ABI against the CPU oracle (pinned by P16): apply, rhs,
forward model and CG on seeded uniform samples, edge positions, every order."""
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
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def dev(a, dt="f64"):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.float64 if dt == "f64" else torch.float32)


def host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy()


def samples(n, K, seed=3):
    """Uniform samples plus the edge cases: corners, integer positions, t = n-1."""
    t = synth.scattered_positions(n, K, seed=seed)
    nn = np.asarray(n, dtype=np.float64)
    extra = [np.zeros(len(n)), nn - 1.0, np.floor(t[0]), np.minimum(np.floor(t[1]) + 1.0, nn - 1.0),
             np.where(np.arange(len(n)) % 2 == 0, 0.0, nn - 1.0)]
    return np.vstack([t] + [e[None, :] for e in extra])


# (n, K, lam): every order, several tiles per mode, ragged tiles, n4 classes,
# a sparse case (many empty tiles) and a dense one (many samples per tile)
CASES = [((12, 11, 10, 16), 3000, 1e-2),
         ((9, 17, 6, 15), 500, 1e-3),
         ((5, 6, 7, 32), 800, 1e-2),
         ((20, 18, 16, 3), 100, 1e-2),
         ((14, 13, 12), 4000, 1e-2),
         ((30, 27), 600, 1e-2),
         ((40,), 70, 1e-1),
         ((8, 8, 8, 8), 20000, 0.0)]
IDS = ["x".join(map(str, c[0])) + f"-K{c[1]}" for c in CASES]


@pytest.mark.parametrize("case", CASES, ids=IDS)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_scattered_apply_rhs_forward_match_oracle(case, dt, tca):
    n, K, lam = case
    t = samples(n, K)
    L = [synth.second_difference(k) for k in n]
    o = oracle.ScatteredOperator(n, t, L, lam)
    g = tca.Operator.scattered(n, t, L, lam, dtype=dt)
    assert g.apply_path == "ksum" and g.Mloc == t.shape[0]
    tol = 1e-12 if dt == "f64" else 1e-5
    x = synth.random_tensor(n, seed=11)
    assert rel(host(g.apply(dev(x, dt))), o.apply(x)) <= tol
    yk = synth.random_tensor((t.shape[0],), seed=12)
    assert rel(host(g.rhs(dev(yk, dt))), o.rhs(yk)) <= tol
    y = host(g.forward_model(dev(x, dt), sigma=0.0))
    assert rel(y, o.forward(x)) <= tol
    g.close()


def test_scattered_full_grid_equals_gridded_operator(tca):
    """GPU scattered operator on the whole Z5 sample grid = GPU gridded operator."""
    n, m = (10, 9, 12, 8), (17, 15, 20, 14)
    A, L = synth.mode_matrices(n, m)
    pos = [synth.sample_positions(nd, md) for nd, md in zip(n, m)]
    t = np.stack(np.meshgrid(*pos, indexing="ij"), axis=-1).reshape(-1, 4)
    gs = tca.Operator.scattered(n, t, L, 1e-2)
    gg = tca.Operator(A, L, 1e-2)
    x = dev(synth.random_tensor(n, seed=13))
    assert rel(host(gs.apply(x)), host(gg.apply(x))) <= 1e-12
    y = synth.random_tensor(m, seed=14)
    assert rel(host(gs.rhs(dev(y.ravel()))), host(gg.rhs(dev(y)))) <= 1e-12
    gs.close()
    gg.close()


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_scattered_cg_matches_oracle(dt, tca):
    n, K, lam = (12, 10, 14, 16), 6000, 1e-2
    t = samples(n, K)
    L = [synth.second_difference(k) for k in n]
    o = oracle.ScatteredOperator(n, t, L, lam)
    g = tca.Operator.scattered(n, t, L, lam, dtype=dt)
    yk = o.forward(synth.random_tensor(n, seed=15)) + 0.01 * synth.random_tensor((t.shape[0],), seed=16)
    b = o.rhs(yk)
    k = 20 if dt == "f32" else 45
    x, rep = g.cg_solve(dev(b, dt), rtol=0.0, max_iters=k)
    xr, kr, st, _ = o.cg(b, rtol=0.0, max_iters=k)
    assert rep["iterations"] == kr == k
    assert rel(host(x), xr) <= (1e-8 if dt == "f64" else 1e-5)
    # single-reduction CG runs on it too (iterates equal to rounding)
    xs, rep2 = g.cgsr_solve(dev(b, dt), rtol=0.0, max_iters=k)
    assert rel(host(xs), xr) <= (1e-7 if dt == "f64" else 1e-4)
    g.close()


def test_scattered_host_solve_and_tolerance_stop(tca):
    n, K, lam = (8, 9, 10, 16), 3000, 1e-2
    t = samples(n, K)
    L = [synth.second_difference(k) for k in n]
    o = oracle.ScatteredOperator(n, t, L, lam)
    g = tca.Operator.scattered(n, t, L, lam)
    yk = o.forward(synth.random_tensor(n, seed=17))
    yh = torch.from_numpy(yk).pin_memory()
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    rep = g.solve_host(yh, xh, rtol=1e-10, max_iters=2000)
    assert rep["converged"]
    xr, kr, st, _ = o.cg(o.rhs(yk), rtol=1e-10, max_iters=2000)
    assert st == oracle.OK and abs(rep["iterations"] - kr) <= 1
    xr, _, _, _ = o.cg(o.rhs(yk), rtol=0.0, max_iters=rep["iterations"])
    assert rel(xh.numpy(), xr) <= 1e-8
    g.close()


def test_scattered_edge_cases(tca):
    n = (6, 7, 8, 5)
    L = [synth.second_difference(k) for k in n]
    # no samples: the regulariser alone
    g = tca.Operator.scattered(n, np.zeros((0, 4)), L, 0.5)
    x = synth.random_tensor(n, seed=18)
    o = oracle.ScatteredOperator(n, np.zeros((0, 4)), L, 0.5)
    assert rel(host(g.apply(dev(x))), o.apply(x)) <= 1e-12
    g.close()
    # one sample, no regulariser: rank-1 operator w w^T
    t = np.array([[2.5, 3.25, 0.0, 4.0]])
    g = tca.Operator.scattered(n, t, None, 0.0)
    o = oracle.ScatteredOperator(n, t, None, 0.0)
    assert rel(host(g.apply(dev(x))), o.apply(x)) <= 1e-12
    g.close()
    # rejected inputs
    for bad in (np.array([[0.0, 0.0, 0.0, 4.5]]), np.array([[-0.1, 0.0, 0.0, 0.0]]),
                np.array([[np.nan, 0.0, 0.0, 0.0]])):
        with pytest.raises(tca.TcaError):
            tca.Operator.scattered(n, bad, L, 0.1)
    g = tca.Operator.scattered(n, samples(n, 50), L, 0.1)
    b = dev(synth.random_tensor(n, seed=19))
    with pytest.raises(tca.TcaError):
        g.pcg_solve(b, max_iters=3)
    with pytest.raises(tca.TcaError):
        g.jacobi_solve(b, max_iters=3)
    g.close()


def test_scattered_paper_grid_sampled(tca):
    """The paper's grid (Sec. 4: 128^3 x 16) with 1e6 samples: apply at sampled
    outputs against the oracle's data term restricted to the samples whose
    support covers them (brute force per output)."""
    n = synth.SCATTER_SHAPE
    K = 1_000_000
    t = synth.scattered_positions(n, K, seed=7)
    L = [synth.second_difference(k) for k in n]
    g = tca.Operator.scattered(n, t, L, 1e-3)
    x = synth.random_tensor(n, seed=20)
    y = host(g.apply(dev(x)))
    rng = np.random.default_rng(2)
    pts = [tuple(int(rng.integers(0, nd)) for nd in n) for _ in range(40)] + [(0, 0, 0, 0), (127, 127, 127, 15)]
    reg = oracle.Operator.from_gram(None, [l.T @ l for l in L], 1e-3).apply(x)
    for p in pts:
        near = np.all(np.abs(t - np.asarray(p)[None, :]) < 2.0, axis=1)   # samples whose w_k touches p
        sub = oracle.ScatteredOperator(n, t[near], None, 0.0)
        want = sub.data(x)[p] + reg[p]
        assert abs(y[p] - want) <= 1e-12 * max(1.0, abs(want))
    g.close()


def test_scattered_host_batch(tca):
    """Pipelined host solves (tca_solve_host_batch) on a scattered operator: K
    sample values per item in, x out; each item equals its single solve."""
    n, K, lam = (8, 7, 9, 16), 2500, 1e-2
    t = samples(n, K)
    L = [synth.second_difference(k) for k in n]
    o = oracle.ScatteredOperator(n, t, L, lam)
    g = tca.Operator.scattered(n, t, L, lam)
    ys = [torch.from_numpy(o.forward(synth.random_tensor(n, seed=s))).contiguous().pin_memory() for s in (21, 22)]
    xs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in ys]
    reps = g.solve_host_batch(ys, xs, rtol=0.0, max_iters=30)
    assert [r["iterations"] for r in reps] == [30, 30]
    for y, x in zip(ys, xs):
        xr, _, _, _ = o.cg(o.rhs(y.numpy()), rtol=0.0, max_iters=30)
        assert rel(x.numpy(), xr) <= 1e-8
    g.close()
