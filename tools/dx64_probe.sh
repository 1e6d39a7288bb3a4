#!/bin/bash
# (experiment record: the variant this measured was reverted; see its log under profiles/ and DESIGN.md 6.3)
# fp64 deferred-x apply (MODE 2 at 112 registers) vs the default iteration, config 3
mkdir -p gpurun_out/dx64
for i in 1 2; do
  TCA_DX=0 python tools/cg_probe.py --dtype f64 --iters 200
  TCA_DX=1 python tools/cg_probe.py --dtype f64 --iters 200
done > gpurun_out/dx64/probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dx.py -m gpu -x -q > gpurun_out/dx64/tests.log 2>&1
cat gpurun_out/dx64/probe.log; tail -3 gpurun_out/dx64/tests.log
