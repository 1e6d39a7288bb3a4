"""Separable Poisson operator (Eq. 9, reading Z25) built from its factors and the
paper's tensor Jacobi solver (Fig. 1, reading Z26) on the GPU, against the
oracle (pinned by P15 in test_oracle_pins.py)."""
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


SHAPES = [(32, 33, 34), (12, 12, 12), (20, 11, 16, 8), (40,), (24, 20)]


@pytest.mark.parametrize("n", SHAPES, ids=["x".join(map(str, n)) for n in SHAPES])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_poisson_apply_matches_oracle(n, dt, tca):
    T = [synth.laplacian_1d(k) for k in n]
    g = tca.Operator.from_gram(None, T, 1.0, dtype=dt)
    assert g.apply_path == "ksum"
    o = oracle.Operator.from_gram(None, T, 1.0)
    x = synth.random_tensor(n, seed=41)
    y = g.apply(dev(x, dt)).double().cpu().numpy()
    assert rel(y, o.apply(x)) <= (1e-12 if dt == "f64" else 1e-5)
    with pytest.raises(Exception):
        g.rhs(dev(x, dt))
    g.close()


def test_gram_form_with_product_term_matches_oracle(tca):
    """Factors given directly, with a Kronecker-product term: same operator as
    the A_d / L_d form."""
    n, m = (24, 11, 36, 15), (48, 22, 72, 30)
    A, L = synth.mode_matrices(n, m, seed=2)
    G = [a.T @ a for a in A]
    R = [l.T @ l for l in L]
    g = tca.Operator.from_gram(G, R, 1e-3)
    assert g.apply_path == "fused"
    x = synth.random_tensor(n, seed=42)
    o = oracle.Operator(A, L, 1e-3)
    assert rel(g.apply(dev(x)).cpu().numpy(), o.apply(x)) <= 1e-12
    g.close()


@pytest.mark.parametrize("n", [(12, 12, 12), (20, 11, 16, 8)])
def test_jacobi_matches_oracle(n, tca):
    T = [synth.laplacian_1d(k) for k in n]
    g = tca.Operator.from_gram(None, T, 1.0)
    o = oracle.Operator.from_gram(None, T, 1.0)
    b = synth.random_tensor(n, seed=43)
    for thr, iters in ((0.0, 7), (0.0, 60), (1e-4, 20000)):   # fixed steps (eager / graph chunks), threshold stop
        u, rep = g.jacobi_solve(dev(b), threshold=thr, max_iters=iters, history=True)
        uo, ko, st, h = o.jacobi(b, threshold=thr, max_iters=iters)
        assert rep["iterations"] == ko
        assert rep["converged"] == (st == oracle.OK)
        assert rel(u.cpu().numpy(), uo) <= 1e-10
        assert np.allclose(rep["rho_history"], h, rtol=1e-8, atol=1e-14 * h[0])
    g.close()


def test_poisson_cg_matches_oracle(tca):
    n = (32, 33, 34)
    T = [synth.laplacian_1d(k) for k in n]
    g = tca.Operator.from_gram(None, T, 1.0)
    o = oracle.Operator.from_gram(None, T, 1.0)
    b = synth.random_tensor(n, seed=44)
    x, rep = g.cg_solve(dev(b), rtol=1e-10, max_iters=2000)
    xo, ko, st, _ = o.cg(b, rtol=0.0, max_iters=rep["iterations"])
    assert rep["converged"] and rel(x.cpu().numpy(), xo) <= 1e-8
    g.close()
