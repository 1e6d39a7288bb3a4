"""PCG probe (not a test): config 3 P^-1 r timing (median of 9 after warm-up, CUDA
events) and time to solution of CG vs PCG at rtol 1e-8 (f64)."""
import os, sys, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1001_5460_b200 import tca

c = synth.CONFIGS[3]
A, L = synth.mode_matrices(c)
for dt in ("f64", "f32"):
    op = tca.Operator(A, L, c.lam, dtype=dt)
    r = torch.empty(op.local_n, dtype=op.torch_dtype, device="cuda")
    tca.generate_normal(r, seed=3, stream_id=7)
    z = torch.empty_like(r)
    for _ in range(3):
        op.precond_apply(r, z)
    ts = []
    for _ in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); op.precond_apply(r, z); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    out = {"dtype": dt, "precond_us": 1e3 * ts[4]}
    y = op.forward_model(None, sigma=synth.NOISE_SIGMA, seed=1)
    b = op.rhs(y)
    del y
    rtol = 1e-8 if dt == "f64" else 1e-5
    for name in ("cg_solve", "pcg_solve"):
        fn = getattr(op, name)
        fn(b, rtol=rtol, max_iters=3)
        x, rep = fn(b, rtol=rtol, max_iters=2000)
        out[name] = {"iters": rep["iterations"], "ms": rep["seconds"] * 1e3, "relres": rep["relres_final"]}
    print(json.dumps(out), flush=True)
    op.close()
