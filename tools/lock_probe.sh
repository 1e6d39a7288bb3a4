#!/bin/bash
# apply schedule (split default vs lock-step, TCA_BAND_SCHED=lock) with the L2 hand-off of the vector kernels
mkdir -p gpurun_out/lock
for i in 1 2 3; do
  for v in split lock; do echo "f64 sched=$v"; TCA_BAND_SCHED=$v python tools/cg_probe.py --dtype f64 --iters 200; done
  for v in split lock; do echo "f32 sched=$v"; TCA_BAND_SCHED=$v python tools/cg_probe.py --dtype f32 --iters 200; done
done > gpurun_out/lock/probe.log 2>&1
cat gpurun_out/lock/probe.log
