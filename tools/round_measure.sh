#!/bin/bash
# One GPU session: bench lines (f64 with cpu baseline, f32), time-to-solution
# table, ncu launch list of the bench command, ncu --set full of the fused apply.
set -u
tag=${1:-v15}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
timeout 400 python bench.py --dtype f32 --no-cpu-baseline > gpurun_out/bench_${tag}_f32.json 2>&1
bash tools/ttsolve.sh gpurun_out/ttsolve_${tag}.txt > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch_${tag}.log 2>&1
for dt in f64 f32; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:band_apply -s 3 -c 1 \
    -o gpurun_out/band_${tag}_${dt} python tools/apply_probe.py --dtype $dt --reps 2 > /dev/null 2>&1
done
tail -c 400 gpurun_out/bench_${tag}.json; echo; tail -c 300 gpurun_out/bench_${tag}_f32.json; echo
cat gpurun_out/ttsolve_${tag}.txt
ls -la gpurun_out/*${tag}*
