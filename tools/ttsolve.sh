#!/bin/bash
# Time to solution, CG vs Kronecker-factor PCG (bench.py --solver), one line per run.
out=${1:-gpurun_out/ttsolve.txt}
: > "$out"
run() {
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
r = d['cg_report']
print(f\"{d['config']['workload']:100s} ttsolve {d['time_to_solution_ms']:9.2f} ms  iters {r['iterations']:4d}  status {r['status']}  it/s {d['value']:9.1f}  rr/rr0 {r['rho_final']/r['rho0']:.2e}\")
" >> "$out"
}
for s in cg pcg; do
  run --config 0 --solver $s
  run --config 1 --solver $s
  run --config 2 --solver $s --rtol 1e-10 --iters 2000
  run --config 3 --solver $s --rtol 1e-10 --iters 2000
  run --config 3 --dtype f32 --solver $s --rtol 1e-6 --iters 2000
done
cat "$out"
