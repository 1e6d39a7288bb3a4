#!/bin/bash
# B1' bring-up: its tests, then CG timing with and without the fused step
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_b1.py -x -q 2>&1 | tail -15
for dt in f64 f32; do
  echo "== $dt B1'"; timeout 120 python tools/apply_probe.py --dtype $dt --reps 10 --cg 100
  echo "== $dt B1' (again)"; timeout 120 python tools/apply_probe.py --dtype $dt --reps 10 --cg 100
  echo "== $dt unfused"; TCA_NO_B1=1 timeout 120 python tools/apply_probe.py --dtype $dt --reps 10 --cg 100
done
