#!/bin/bash
# (experiment record: the variant this measured was reverted; see profiles/r02_xp_grid_probe.txt)
# (experiment) cg_update_xp grid: 592 CTAs (default) vs 2x / 4x
mkdir -p gpurun_out/xpg
for i in 1 2 3; do
  for v in 1 2 4; do echo "f64 TCA_XP_GRID=$v"; TCA_XP_GRID=$v python tools/cg_probe.py --dtype f64 --iters 200; done
done > gpurun_out/xpg/probe.log 2>&1
cat gpurun_out/xpg/probe.log
