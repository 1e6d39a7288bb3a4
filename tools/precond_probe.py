"""Time z = P^-1 r (PCG preconditioner) for a config; for ncu launch lists."""
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
a = ap.parse_args()
c = synth.CONFIGS[a.config]
A, L = synth.mode_matrices(c)
op = tca.Operator(A, L, c.lam, dtype=a.dtype)
tdt = torch.float64 if a.dtype == "f64" else torch.float32
r = torch.empty(c.n, dtype=tdt, device="cuda")
tca.generate_normal(r, seed=3, stream_id=7)
z = torch.empty_like(r)
for _ in range(3):
    op.precond_apply(r, z)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    op.precond_apply(r, z)
e1.record()
torch.cuda.synchronize()
us = 1e3 * e0.elapsed_time(e1) / a.reps
esize = 8 if a.dtype == "f64" else 4
print(f"config {a.config} {a.dtype}: P^-1 r {us:.1f} us ({2 * c.N * esize / us / 1e3:.0f} GB/s at 2 words)")
