#!/bin/bash
# closing ncu --set full of the fused apply inside CG (f64 and f32) and the launch list of one bench step
mkdir -p gpurun_out/r02n
ncu --set full --import-source on --clock-control none -k regex:band_apply_kernel -s 40 -c 1 \
    -o gpurun_out/r02n/band_f64 \
    python bench.py --steps 1 --warmup 3 --cfg4-iters 0 --small-iters 0 --no-e2e --no-cpu-baseline --apply-reps 5 \
    > gpurun_out/r02n/ncu_full_f64.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:band_apply_kernel -s 40 -c 1 \
    -o gpurun_out/r02n/band_f32 \
    python bench.py --dtype f32 --steps 1 --warmup 3 --cfg4-iters 0 --small-iters 0 --no-e2e --no-cpu-baseline --apply-reps 5 \
    > gpurun_out/r02n/ncu_full_f32.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/r02n/launches_f64.csv \
    python bench.py --steps 1 --warmup 3 --cfg4-iters 0 --small-iters 0 --no-e2e --no-cpu-baseline --apply-reps 5 \
    > gpurun_out/r02n/ncu_launch.log 2>&1
ls gpurun_out/r02n
