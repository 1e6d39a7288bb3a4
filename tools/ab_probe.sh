#!/bin/bash
# A/B timing of library variants in one GPU session: tools/ab_probe.sh lib1.so lib2.so ...
for lib in "$@"; do
  cp "$lib" paper_1001_5460_b200/libtca.so
  for rep in 1 2; do
    echo "== $lib (rep $rep)"
    timeout 60 python tools/apply_probe.py --config 3 --dtype f64 --reps 30 --cg 30
  done
done
