#!/bin/bash
# one ncu --set full capture (with source) of the fused apply: tools/ncu_full.sh NAME [dtype] [extra env]
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:band_apply_kernel -s 5 -c 1 \
    -o gpurun_out/$1 python tools/apply_probe.py --dtype ${2:-f64} --reps 3 > gpurun_out/$1.log 2>&1
