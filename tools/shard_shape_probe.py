"""Apply time on the per-GPU shapes of config 3 sharded over P = 8/4/2/1 GPUs (mode-1 rows 16..128)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_1001_5460_b200 import tca
# per-GPU shape of config 3 on P = 8 / 4 / 2 / 1 (mode-1 rows 16 / 32 / 64 / 128)
for n1 in (16, 32, 64, 128):
    n, m = (n1, 128, 128, 15), (2 * n1, 256, 256, 30)
    A, L = synth.mode_matrices(n, m)
    op = tca.Operator(A, L, 1e-3)
    x = torch.empty(n, dtype=torch.float64, device="cuda"); tca.generate_normal(x, seed=3, stream_id=7)
    y = torch.empty_like(x)
    for _ in range(3): op.apply(x, y)
    op.set_timing(True)
    for _ in range(20): op.apply(x, y)
    ms, cnt = op.get_timing()
    print(f"n1={n1}: {1e3*ms/cnt:.1f} us ({1e3*ms/cnt/n1:.2f} us per mode-1 row)")
    op.close()
