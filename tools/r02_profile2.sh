#!/bin/bash
# Round-2 evidence run (one GPU): bench lines (f64 default, f32, pcg), the ncu
# launch list of one bench step, one ncu --set full capture of the fused apply
# (fp64 and fp32), all under gpurun_out/r02h/.
set -x
mkdir -p gpurun_out/r02h
python bench.py > gpurun_out/r02h/bench_f64.log 2>&1
python bench.py --dtype f32 --cfg4-iters 0 --small-iters 0 > gpurun_out/r02h/bench_f32.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/r02h/launches_f64.csv \
    python bench.py --steps 1 --warmup 3 --cfg4-iters 0 --small-iters 0 --no-e2e --no-cpu-baseline --apply-reps 5 \
    > gpurun_out/r02h/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:band_apply_kernel -s 40 -c 1 \
    -o gpurun_out/r02h/band_f64 \
    python bench.py --steps 1 --warmup 3 --cfg4-iters 0 --small-iters 0 --no-e2e --no-cpu-baseline --apply-reps 5 \
    > gpurun_out/r02h/ncu_full_f64.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:band_apply_kernel -s 40 -c 1 \
    -o gpurun_out/r02h/band_f32 \
    python bench.py --dtype f32 --steps 1 --warmup 3 --cfg4-iters 0 --small-iters 0 --no-e2e --no-cpu-baseline --apply-reps 5 \
    > gpurun_out/r02h/ncu_full_f32.log 2>&1
tail -c 400 gpurun_out/r02h/bench_f64.log
