#!/bin/bash
# A/B timing (fp32, config 3) of library variants in one GPU session
for lib in "$@"; do
  cp "$lib" paper_1001_5460_b200/libtca.so
  echo "== $lib"
  timeout 60 python tools/apply_probe.py --config 3 --dtype f32 --reps 30 --cg 30
done
