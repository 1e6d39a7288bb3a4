"""Time the standalone operator apply for a config (for ncu captures)."""
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
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--cg", type=int, default=0, help="also run this many CG iterations")
ap.add_argument("--only-cg", action="store_true", help="skip the standalone applies (ncu of the CG kernels)")
args = ap.parse_args()
c = synth.CONFIGS[args.config]
A, L = synth.mode_matrices(c)
op = tca.Operator(A, L, c.lam, dtype=args.dtype)
tdt = torch.float64 if args.dtype == "f64" else torch.float32
x = torch.empty(c.n, dtype=tdt, device="cuda")
tca.generate_normal(x, seed=3, stream_id=7)
y = torch.empty_like(x)
for _ in range(0 if args.only_cg else 3):
    op.apply(x, y)
torch.cuda.synchronize()
op.set_timing(True)
for _ in range(0 if args.only_cg else args.reps):
    op.apply(x, y)
torch.cuda.synchronize()
ms, cnt = op.get_timing()
esize = 8 if args.dtype == "f64" else 4
if cnt:
    us = 1e3 * ms / cnt
    print(f"config {args.config} {args.dtype}: apply {us:.1f} us, {2*c.N*esize/us/1e3:.1f} GB/s")
if args.cg:
    xs, rep = op.cg_solve(x, rtol=0.0, max_iters=args.cg)
    ms, cnt = op.get_timing()
    print(f"CG {rep['iterations']} it: {rep['seconds']*1e3:.2f} ms, apply in CG {1e3*ms/max(cnt,1):.1f} us")
