#!/bin/bash
# A/B of two library builds on the config-3 fp32 apply (tools/scratch/*.so)
for lib in "$@" "$@"; do
  cp $lib paper_1001_5460_b200/libtca.so
  echo "== $lib"; timeout 60 python tools/apply_probe.py --dtype f32 --reps 30 --cg 30 2>&1 | tail -2
done
