#!/bin/bash
# finalisers fused into their producer kernels (tca_finalize.cuh) vs the
# separate finaliser kernels (TCA_NO_FUSED_FIN=1): config 3 CG per iteration, then the GPU suite
mkdir -p gpurun_out/fin
for i in 1 2; do
  for dt in f64 f32; do
    TCA_NO_FUSED_FIN=1 python tools/cg_probe.py --dtype $dt --iters 200
    python tools/cg_probe.py --dtype $dt --iters 200
  done
done > gpurun_out/fin/probe.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin/gputest.log 2>&1
cat gpurun_out/fin/probe.log; tail -3 gpurun_out/fin/gputest.log
