#!/bin/bash
# (experiment record: the variant this measured was reverted; see its log under profiles/ and DESIGN.md 6.3)
# deferred x update over a ring of P buffers (TCA_XD=0|2|4) and programmatic
# dependent launch (TCA_PDL=0|1): config 3 CG per iteration, the XD tests, then
# the full GPU suite
mkdir -p gpurun_out/xd
timeout 900 python -m pytest tests/test_gpu_xd.py -x -q > gpurun_out/xd/xdtest.log 2>&1
tail -3 gpurun_out/xd/xdtest.log
for i in 1 2; do
  for cfg in "0 0" "0 1" "4 0" "4 1" "2 1"; do
    set -- $cfg
    echo "f64 TCA_XD=$1 TCA_PDL=$2"; TCA_XD=$1 TCA_PDL=$2 python tools/cg_probe.py --dtype f64 --iters 200
  done
  echo "f32 DX PDL=0"; TCA_PDL=0 python tools/cg_probe.py --dtype f32 --iters 200
  echo "f32 DX PDL=1"; TCA_PDL=1 python tools/cg_probe.py --dtype f32 --iters 200
  echo "f32 DX=0 XD=4 PDL=1"; TCA_DX=0 TCA_XD=4 python tools/cg_probe.py --dtype f32 --iters 200
done > gpurun_out/xd/probe.log 2>&1
cat gpurun_out/xd/probe.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/xd/gputest.log 2>&1
tail -3 gpurun_out/xd/gputest.log
