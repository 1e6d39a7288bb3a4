"""CG time per iteration on config 3 (fixed iterations, device-resident): python tools/cg_probe.py [--dtype f64] [--iters 200]."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1001_5460_b200 import tca  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--dtype", default="f64")
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--solver", default="cg")
args = ap.parse_args()
c = synth.CONFIGS[args.config]
A, L = synth.mode_matrices(c)
op = tca.Operator(A, L, c.lam, dtype=args.dtype)
tdt = torch.float64 if args.dtype == "f64" else torch.float32
b = torch.empty(c.n, dtype=tdt, device="cuda")
tca.generate_normal(b, seed=3, stream_id=7)
solve = op.pcg_solve if args.solver == "pcg" else op.cg_solve
solve(b, rtol=0.0, max_iters=40)
torch.cuda.synchronize()
best = None
for rep in range(3):
    x, r = solve(b, rtol=0.0, max_iters=args.iters)
    us = r["seconds"] * 1e6 / r["iterations"]
    best = us if best is None else min(best, us)
op.set_timing(True)
x, r = solve(b, rtol=0.0, max_iters=args.iters)
ms, cnt = op.get_timing()
print(f"config {args.config} {args.dtype} {args.solver}: {best:.1f} us per iteration (best of 3, {r['iterations']} it), "
      f"apply in CG {1e3 * ms / max(cnt, 1):.1f} us, rho_final {r['rho_final']:.3e} relres {r['relres_final']:.3e}")
