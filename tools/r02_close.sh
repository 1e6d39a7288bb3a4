#!/bin/bash
# closing check at HEAD: GPU suite, smoke, bench lines
mkdir -p gpurun_out/r02d
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02d/gputest.log 2>&1
tail -3 gpurun_out/r02d/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d/smoke.log 2>&1; tail -1 gpurun_out/r02d/smoke.log
python bench.py > gpurun_out/r02d/bench_f64.log 2>&1
python bench.py --dtype f32 --cfg4-iters 0 > gpurun_out/r02d/bench_f32.log 2>&1
tail -c 400 gpurun_out/r02d/bench_f64.log
