"""Grid-engine probe (not a test): us per CG iteration on configs 1 and 2 (f64),
200 fixed iterations, best of 3; run with TCA_GRID_DBG=1/2/3 to drop phases."""
import os, sys, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1001_5460_b200 import tca
out = {"dbg": os.environ.get("TCA_GRID_DBG", "0")}
for ci in (1, 2):
    c = synth.CONFIGS[ci]
    A, L = synth.mode_matrices(c)
    op = tca.Operator(A, L, c.lam)
    b = op.rhs(torch.from_numpy(synth.data(A, c.n, c.m, seed=1)).cuda())
    op.cg_solve(b, rtol=0.0, max_iters=10)
    best = min(op.cg_solve(b, rtol=0.0, max_iters=200)[1]["seconds"] for _ in range(3))
    out[f"config{ci}"] = {"engine": op.cg_engine, "us_per_it": best * 1e6 / 200}
    op.close()
print(json.dumps(out))
