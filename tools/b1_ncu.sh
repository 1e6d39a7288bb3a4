#!/bin/bash
set -u
mkdir -p gpurun_out
tag=${1:-x}
timeout 900 python -m pytest tests/test_gpu_b1.py -x -q 2>&1 | tail -4
for dt in f64 f32; do
  echo "== $dt B1'"; timeout 120 python tools/apply_probe.py --dtype $dt --reps 10 --cg 100
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:band_apply -s 3 -c 1 \
  -o gpurun_out/b1_${tag}_f64 python tools/apply_probe.py --dtype f64 --only-cg --cg 8 > gpurun_out/b1_ncu.log 2>&1
