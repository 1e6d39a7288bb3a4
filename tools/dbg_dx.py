import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_1001_5460_b200 import tca
n, m, lam = (32, 32, 30, 15), (64, 64, 60, 30), 1e-2
A, L = synth.mode_matrices(n, m, seed=2)
b = synth.random_tensor(n, seed=6)
for dt in ("f32", "f64"):
    for k in (1, 2, 20):
        os.environ["TCA_DX"] = "1"
        op = tca.Operator(A, L, lam, dtype=dt)
        tdt = torch.float32 if dt == "f32" else torch.float64
        x, rep = op.cg_solve(torch.from_numpy(b).cuda().to(tdt), rtol=0.0, max_iters=k)
        print(dt, k, "dx", op.cg_deferred_x, "b1", op.cg_fused_step, "path", op.apply_path, "engine", tca._lib.tca_operator_cg_engine(op._h))
        op.close()
