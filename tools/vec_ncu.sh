#!/bin/bash
# DRAM bytes and time of the CG vector kernels inside the solve, caches NOT flushed between
# kernels (so the L2 hand-off shows), default vs TCA_L2REV=0
mkdir -p gpurun_out/vecncu
for v in 1 0; do
  TCA_L2REV=$v ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:"cg_update|band_apply" -s 300 -c 12 --csv python tools/cg_probe.py --dtype f64 --iters 60 > gpurun_out/vecncu/l2rev$v.csv 2>&1
done
tail -5 gpurun_out/vecncu/l2rev1.csv
