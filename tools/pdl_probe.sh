#!/bin/bash
# (experiment record: the variant this measured was reverted; see its log under profiles/ and DESIGN.md 6.3)
# programmatic dependent launch of the CG kernel chain vs plain launches (TCA_PDL=0): config 3
# CG per iteration; then the GPU parity suite and the f64 bench line
mkdir -p gpurun_out/pdl
for i in 1 2; do
  for dt in f64 f32; do
    TCA_PDL=0 python tools/cg_probe.py --dtype $dt --iters 200
    python tools/cg_probe.py --dtype $dt --iters 200
  done
done > gpurun_out/pdl/probe.log 2>&1
cat gpurun_out/pdl/probe.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pdl/gputest.log 2>&1
tail -3 gpurun_out/pdl/gputest.log
python bench.py > gpurun_out/pdl/bench_f64.log 2>&1; tail -c 600 gpurun_out/pdl/bench_f64.log
