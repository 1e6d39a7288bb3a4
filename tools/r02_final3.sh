#!/bin/bash
# closing round-2 evidence at HEAD: bench lines (f64 default, f32), the launch list of one f64 step
mkdir -p gpurun_out/r02z
python bench.py > gpurun_out/r02z/bench_f64.log 2>&1
python bench.py --dtype f32 --cfg4-iters 0 > gpurun_out/r02z/bench_f32.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/r02z/launches_f64.csv \
    python bench.py --steps 1 --warmup 3 --cfg4-iters 0 --small-iters 0 --no-e2e --no-cpu-baseline --apply-reps 5 \
    > gpurun_out/r02z/ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z/smoke.log 2>&1
tail -c 300 gpurun_out/r02z/bench_f64.log; tail -2 gpurun_out/r02z/smoke.log
