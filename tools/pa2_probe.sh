#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "apply" 2>&1 | tail -2
for lib in tools/scratch/base.so tools/scratch/pa2.so tools/scratch/base.so tools/scratch/pa2.so; do
  cp $lib paper_1001_5460_b200/libtca.so
  for dt in f64 f32; do echo "== $lib $dt"; timeout 60 python tools/apply_probe.py --dtype $dt --reps 30 --cg 30 2>&1 | tail -2; done
done
cp tools/scratch/pa2.so paper_1001_5460_b200/libtca.so
