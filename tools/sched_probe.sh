#!/bin/bash
# Schedule A/B (config 3): apply standalone and in CG, DRAM bytes per launch (ncu).
set -u
for sch in ${SCHEDS:-split lock whole}; do
 for dt in ${DTYPES:-f64 f32}; do
  echo "== $sch $dt"
  TCA_BAND_SCHED=$sch timeout 120 python tools/apply_probe.py --dtype $dt --reps 30 --cg 30
  TCA_BAND_SCHED=$sch timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:band_apply -s 3 -c 1 python tools/apply_probe.py --dtype $dt --reps 2 2>&1 | grep -E "dram__|lts__|gpu__time"
 done
done
