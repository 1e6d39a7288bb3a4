"""Phase timing of tca_solve_host on config 3 (H2D, rhs+CG, D2H)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1001_5460_b200 import tca
c = synth.CONFIGS[3]
A, L = synth.mode_matrices(c)
op = tca.Operator(A, L, c.lam, dtype="f64")
yd = op.forward_model(None, sigma=0.01, seed=1)
yh = torch.empty(yd.shape, dtype=torch.float64, pin_memory=True); yh.copy_(yd.cpu())
xh = torch.empty(c.n, dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()
for it in range(3):
    t0 = time.perf_counter()
    ydev = torch.empty_like(yd)
    ydev.copy_(yh, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter()
    rep = op.solve_host(yh, xh, rtol=0.0, max_iters=500)
    t2 = time.perf_counter()
    print(f"h2d alone {1e3*(t1-t0):.1f} ms ({yh.numel()*8/(t1-t0)/1e9:.1f} GB/s); solve_host {1e3*(t2-t1):.1f} ms (cg {rep['seconds']*1e3:.1f} ms)")
op.close()
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = tca.Operator(A, L, c.lam, dtype="f64")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rep = op.solve_host(yh, xh, rtol=0.0, max_iters=500)
    t2 = time.perf_counter()
    op.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms, solve_host {1e3*(t2-t1):.1f} ms, close {1e3*(t3-t2):.1f} ms")
