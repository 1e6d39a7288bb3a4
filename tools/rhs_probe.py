"""rhs timing probe (not a test): config 3 (and 4 with --cfg4) b = (kron A_d^T) y,
median of 5 timed calls after 2 warm-ups, CUDA events on the current stream."""
import os, sys, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1001_5460_b200 import tca

def probe(ci, dtype):
    c = synth.CONFIGS[ci]
    A, L = synth.mode_matrices(c)
    op = tca.Operator(A, L, c.lam, dtype=dtype)
    y = op.forward_model(None, sigma=synth.NOISE_SIGMA, seed=1)
    ts = []
    for i in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b = op.rhs(y); e1.record(); torch.cuda.synchronize()
        if i >= 2: ts.append(e0.elapsed_time(e1))
        del b
    ts.sort()
    nbytes = (y.numel() + op.N) * y.element_size()
    op.close(); del y; torch.cuda.empty_cache()
    return {"config": ci, "dtype": dtype, "rhs_ms": ts[len(ts) // 2], "floor_ms": nbytes / 6548.5e9 * 1e3}

cfgs = [3] + ([4] if "--cfg4" in sys.argv else [])
for ci in cfgs:
    for dt in ("f64", "f32"):
        print(json.dumps(probe(ci, dt)), flush=True)
