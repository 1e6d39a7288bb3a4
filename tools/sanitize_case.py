"""Small fused-apply / CG / sharded run for compute-sanitizer (memcheck / racecheck)."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1001_5460_b200 import tca
for n, m in [((13, 11, 36, 15), (26, 22, 72, 30)), ((12, 12, 12), (20, 20, 20)), ((9, 70, 16, 7), (18, 140, 32, 14))]:
    A, L = synth.mode_matrices(n, m)
    for dt in ("f64", "f32"):
        op = tca.Operator(A, L, 1e-3, dtype=dt)
        x = torch.empty(op.local_n, dtype=op.torch_dtype, device="cuda")
        tca.generate_normal(x, seed=3, stream_id=7)
        y = op.apply(x)
        yd = op.forward_model(None, sigma=0.01, seed=1)
        b = op.rhs(yd)
        xs, rep = op.cg_solve(b, rtol=0.0, max_iters=40)
        torch.cuda.synchronize()
        print(n, dt, op.apply_path, rep["iterations"], flush=True)
        op.close()
print("done")
