"""One config-1 grid-engine solve (for ncu captures)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1001_5460_b200 import tca
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = synth.CONFIGS[ci]
A, L = synth.mode_matrices(c)
op = tca.Operator(A, L, c.lam)
b = op.rhs(torch.from_numpy(synth.data(A, c.n, c.m, seed=1)).cuda())
op.cg_solve(b, rtol=0.0, max_iters=50)
torch.cuda.synchronize()
