#!/bin/bash
# L2 hand-off between cg_update_r (reverse sweep) and cg_update_xp (TCA_L2REV=1) vs the streaming default
mkdir -p gpurun_out/l2rev
for i in 1 2 3; do
  for v in 0 1; do echo "f64 TCA_L2REV=$v"; TCA_L2REV=$v python tools/cg_probe.py --dtype f64 --iters 200; done
  for v in 0 1; do echo "f32 TCA_L2REV=$v"; TCA_L2REV=$v python tools/cg_probe.py --dtype f32 --iters 200; done
done > gpurun_out/l2rev/probe.log 2>&1
cat gpurun_out/l2rev/probe.log
