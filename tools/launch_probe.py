"""Host-side launch cost vs device time of the fused apply (config 3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1001_5460_b200 import tca
c = synth.CONFIGS[3]
A, L = synth.mode_matrices(c)
op = tca.Operator(A, L, c.lam, dtype="f64")
x = torch.empty(c.n, dtype=torch.float64, device="cuda"); tca.generate_normal(x, seed=3, stream_id=7)
y = torch.empty_like(x)
for _ in range(3): op.apply(x, y)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50): op.apply(x, y)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host per launch {1e6*(t1-t0)/50:.1f} us, wall per apply {1e6*(t2-t0)/50:.1f} us")
xs, rep = op.cg_solve(x, rtol=0.0, max_iters=50)
print(f"CG 50 it: {rep['seconds']*1e3:.2f} ms -> {rep['seconds']*1e6/50:.1f} us/iteration")
op.set_timing(True)
xs, rep = op.cg_solve(x, rtol=0.0, max_iters=50)
ms, cnt = op.get_timing()
print(f"timed CG 50 it: {rep['seconds']*1e3:.2f} ms, apply in CG {1e3*ms/cnt:.1f} us")
