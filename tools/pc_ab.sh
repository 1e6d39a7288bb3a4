#!/bin/bash
for lib in tools/scratch/base.so tools/scratch/lb64.so tools/scratch/base.so tools/scratch/lb64.so; do
  cp $lib paper_1001_5460_b200/libtca.so
  echo "== $lib"; timeout 60 python tools/precond_probe.py --dtype f64 2>&1 | tail -1; timeout 60 python tools/precond_probe.py --dtype f32 2>&1 | tail -1
done
cp tools/scratch/lb64.so paper_1001_5460_b200/libtca.so
