"""Scattered-data operator at the paper's Sec. 4 size: create, apply, rhs, forward, CG timings."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1001_5460_b200 import tca  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=synth.SCATTER_K)
ap.add_argument("--dtype", default="f64")
ap.add_argument("--cg", type=int, default=50)
args = ap.parse_args()
n = synth.SCATTER_SHAPE
t = synth.scattered_positions(n, args.K, seed=1)
L = [synth.second_difference(k) for k in n]
t0 = time.perf_counter()
op = tca.Operator.scattered(n, t, L, 1e-3, dtype=args.dtype)
torch.cuda.synchronize()
print(f"create {1e3 * (time.perf_counter() - t0):.1f} ms  K={args.K}")
tdt = torch.float64 if args.dtype == "f64" else torch.float32
x = torch.empty(n, dtype=tdt, device="cuda")
tca.generate_normal(x, seed=3, stream_id=7)
y = op.apply(x)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


ms = timeit(lambda: op.apply(x, y))
print(f"apply {ms * 1e3:.1f} us  ({ms * 1e6 / args.K:.2f} ns/sample)")
yk = op.forward_model(x, sigma=0.01)
ms = timeit(lambda: op.forward_model(x, yk, sigma=0.0))
print(f"forward {ms * 1e3:.1f} us")
b = op.rhs(yk)
ms = timeit(lambda: op.rhs(yk, b))
print(f"rhs {ms * 1e3:.1f} us")
op.set_timing(True)
xs, rep = op.cg_solve(b, rtol=0.0, max_iters=args.cg)
ams, cnt = op.get_timing()
print(f"CG {rep['iterations']} it: {rep['seconds'] * 1e3:.1f} ms ({rep['seconds'] * 1e6 / max(1, rep['iterations']):.0f} us/it), apply in CG {1e3 * ams / max(cnt, 1):.1f} us")
