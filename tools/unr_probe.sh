#!/bin/bash
# (experiment) vector kernels with more loads in flight per thread: TCA_L2REV=2 (cg_update_r 4 vectors
# in flight), 3 (and cg_update_xp 2 vectors in flight) vs the default (1)
mkdir -p gpurun_out/unr2
for i in 1 2 3; do
  for v in 1 2 3; do echo "f64 TCA_L2REV=$v"; TCA_L2REV=$v python tools/cg_probe.py --dtype f64 --iters 200; done
  for v in 1 2; do echo "f32 TCA_L2REV=$v"; TCA_L2REV=$v python tools/cg_probe.py --dtype f32 --iters 200; done
done > gpurun_out/unr2/probe.log 2>&1
cat gpurun_out/unr2/probe.log
