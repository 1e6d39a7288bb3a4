#!/bin/bash
# Round-2 bench lines for the secondary workloads (one GPU), under gpurun_out/r02/.
mkdir -p gpurun_out/r02
python bench.py --workload poisson --solver jacobi --steps 3 > gpurun_out/r02/bench_poisson_jacobi.log 2>&1
python bench.py --workload poisson --solver cg --steps 3 > gpurun_out/r02/bench_poisson_cg.log 2>&1
python bench.py --workload scattered --steps 3 > gpurun_out/r02/bench_scattered_f64.log 2>&1
python bench.py --workload scattered --dtype f32 --steps 3 > gpurun_out/r02/bench_scattered_f32.log 2>&1
python bench.py --solver cgsr --steps 3 --cfg4-iters 0 --small-iters 0 --no-e2e > gpurun_out/r02/bench_cgsr.log 2>&1
python bench.py --config 1 --solver pcg --steps 3 --cfg4-iters 0 --small-iters 0 --no-e2e > gpurun_out/r02/bench_pcg_cfg1.log 2>&1
python bench.py --config 1 --steps 3 --cfg4-iters 0 --small-iters 0 --no-e2e > gpurun_out/r02/bench_cg_cfg1.log 2>&1
python tools/dense_probe.py > gpurun_out/r02/dense_probe.log 2>&1
python tools/grid_probe.py > gpurun_out/r02/grid_probe.log 2>&1
python tools/rhs_probe.py --cfg4 > gpurun_out/r02/rhs_probe.log 2>&1
python tools/pcg_probe.py > gpurun_out/r02/pcg_probe.log 2>&1
for f in gpurun_out/r02/bench_*.log; do echo "$f: $(grep -c '^{' $f) line(s)"; done
