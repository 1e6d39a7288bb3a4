"""Diagnostic (not a test): relative error of CG iterates against the oracle per k
for a few small shapes, on whichever engine TCA_TINY selects."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, synth
from paper_1001_5460_b200 import tca
for n, m, basis in [((9, 7, 6, 5), (14, 12, 10, 9), "bspline"), ((11, 10, 9), (16, 15, 14), "gauss")]:
    A, L = synth.mode_matrices(n, m, basis=basis)
    o = oracle.Operator(A, L, 0.01)
    b = o.rhs(synth.data(A, n, m, seed=1))
    for dt in ("f64", "f32"):
        g = tca.Operator(A, L, 0.01, dtype=dt)
        tdt = torch.float64 if dt == "f64" else torch.float32
        out = []
        for k in (1, 2, 3, 5, 10, 20, 30):
            xg, rep = g.cg_solve(torch.from_numpy(b).to("cuda", tdt), rtol=0.0, max_iters=k)
            xo, _, _, h = o.cg(b, rtol=0.0, max_iters=k)
            out.append("k=%d %.1e (rho %.1e)" % (k, np.linalg.norm(xg.double().cpu().numpy() - xo) / np.linalg.norm(xo), h[k] / h[0]))
        print(basis, n, dt, "tiny" if g.tiny_engine else "general", "; ".join(out))
        y = g.apply(torch.from_numpy(b).to("cuda", tdt))
        print("   apply relerr %.1e" % (np.linalg.norm(y.double().cpu().numpy() - o.apply(b)) / np.linalg.norm(o.apply(b))))
