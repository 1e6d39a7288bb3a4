"""Dense-mode apply (Gaussian A_d: the FP64 tensor-core mode products) at 128^3
(tensor-pipe utilisation on a standalone larger dense apply)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1001_5460_b200 import tca  # noqa: E402

n, m = (128, 128, 128), (160, 160, 160)
A, L = synth.mode_matrices(n, m, basis="gauss", seed=1)
op = tca.Operator(A, L, 1e-3)
x = torch.empty(n, dtype=torch.float64, device="cuda")
tca.generate_normal(x, seed=3, stream_id=7)
y = op.apply(x)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
for _ in range(20):
    op.apply(x, y)
e[1].record()
torch.cuda.synchronize()
us = e[0].elapsed_time(e[1]) * 1e3 / 20
N = 128 ** 3
flops = 2 * 3 * 128 * N   # three dense 128 x 128 mode products (Kronecker term)
print(f"dense 128^3 apply ({op.apply_path}): {us:.1f} us, Kronecker-term {flops / us / 1e6:.2f} TFLOP/s fp64")
