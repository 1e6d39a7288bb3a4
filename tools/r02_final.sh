#!/bin/bash
# Final round-2 bench lines (f64 default, f32) and the launch list of the f64 step, under gpurun_out/r02f/.
mkdir -p gpurun_out/r02f
python bench.py > gpurun_out/r02f/bench_f64.log 2>&1
python bench.py --dtype f32 --cfg4-iters 0 > gpurun_out/r02f/bench_f32.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/r02f/launches_f64.csv \
    python bench.py --steps 1 --warmup 3 --cfg4-iters 0 --small-iters 20 --no-e2e --no-cpu-baseline --apply-reps 5 \
    > gpurun_out/r02f/ncu_launch.log 2>&1
tail -c 300 gpurun_out/r02f/bench_f64.log
