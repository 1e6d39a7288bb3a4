#!/bin/bash
# (experiment) vectors in flight per thread in cg_update_r's reverse sweep: library variants built with -DTCA_R_UNR=2|4|8
mkdir -p gpurun_out/runr
cp paper_1001_5460_b200/libtca.so /tmp/libtca_keep.so
for i in 1 2 3; do
  for u in 2 4 8; do
    cp tools/scratch/lib_u$u.so paper_1001_5460_b200/libtca.so
    echo "f64 unroll $u"; python tools/cg_probe.py --dtype f64 --iters 200
  done
done > gpurun_out/runr/probe.log 2>&1
cp /tmp/libtca_keep.so paper_1001_5460_b200/libtca.so
cat gpurun_out/runr/probe.log
