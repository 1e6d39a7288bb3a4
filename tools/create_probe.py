"""Host-side cost of tca_operator_create at a config (operators kept alive, or closed)."""
import argparse
import time

import torch

import synth
from paper_1001_5460_b200 import tca

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--dtype", default="f64")
ap.add_argument("--n", type=int, default=6)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
A, L = synth.mode_matrices(cfg)
keep = []
for mode in ("keep", "close"):
    for i in range(a.n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op = tca.Operator(A, L, cfg.lam, dtype=a.dtype)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if mode == "keep":
            keep.append(op)
        else:
            op.close()
        t2 = time.perf_counter()
        print(f"{mode} {i}: create {1e3 * (t1 - t0):.1f} ms, close {1e3 * (t2 - t1):.1f} ms", flush=True)
    for o in keep:
        o.close()
    keep.clear()
