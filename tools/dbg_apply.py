import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch, synth, oracle
from paper_1001_5460_b200 import tca
def rel(a, b): return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
for (n, m) in [((12,12,12),(20,20,20)), ((13,11,36,15),(26,22,72,30))]:
    A, L = synth.mode_matrices(n, m, basis='bspline', seed=1)
    x = synth.random_tensor(n, seed=5)
    xt = torch.from_numpy(x).cuda()
    for lam in (0.0, 1.0):
        g = tca.Operator(A, L, lam, dtype='f64'); o = oracle.Operator(A, L, lam)
        print(n, 'lam', lam, 'all-modes relerr', rel(g.apply(xt).cpu().numpy(), o.apply(x)), flush=True)
    D = len(n)
    for d in range(D):
        Ls = [L[e] if e == d else None for e in range(D)]
        g = tca.Operator(A, Ls, 1.0, dtype='f64'); o = oracle.Operator(A, Ls, 1.0)
        y = g.apply(xt).cpu().numpy(); r = o.apply(x)
        o0 = oracle.Operator(A, None, 0.0).apply(x)
        print(n, 'reg only mode', d, 'relerr', rel(y, r), 'reg-part relerr', rel(y - o0, r - o0), flush=True)
