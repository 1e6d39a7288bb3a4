#!/bin/bash
# (experiment) cg_update_p (fp32 deferred-x path) with 4 vectors in flight and D read L2-normal vs before
mkdir -p gpurun_out/up
cp paper_1001_5460_b200/libtca.so /tmp/libtca_keep.so
for i in 1 2 3; do
  for v in base up; do
    cp tools/scratch/lib_$v.so paper_1001_5460_b200/libtca.so
    echo "f32 $v"; python tools/cg_probe.py --dtype f32 --iters 200
  done
done > gpurun_out/up/probe.log 2>&1
cp /tmp/libtca_keep.so paper_1001_5460_b200/libtca.so
timeout 600 python -m pytest tests/test_gpu_dx.py -x -q > gpurun_out/up/dxtest.log 2>&1
cat gpurun_out/up/probe.log; tail -2 gpurun_out/up/dxtest.log
