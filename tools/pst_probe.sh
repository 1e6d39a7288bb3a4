#!/bin/bash
# (experiment record: the variant this measured was reverted; see profiles/r02_pstore_probe.txt)
# cg_update_xp storing P L2-normal (TCA_L2REV=3) vs evict-first (1, default)
mkdir -p gpurun_out/pst
for i in 1 2 3; do
  for v in 1 3; do echo "f64 TCA_L2REV=$v"; TCA_L2REV=$v python tools/cg_probe.py --dtype f64 --iters 200; done
done > gpurun_out/pst/probe.log 2>&1
cat gpurun_out/pst/probe.log
