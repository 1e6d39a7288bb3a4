#!/bin/bash
# B1' (opt-in fused CG step) phase costs via TCA_BAND_DEBUG switches (results invalid): config 3 CG step
for d in 0 1 512 1024 2048 3585; do
  echo "== B1' dbg $d"; TCA_B1=1 TCA_BAND_DEBUG=$d timeout 120 python tools/apply_probe.py --dtype f64 --only-cg --cg 100 2>&1 | tail -1
done
echo "== unfused"; timeout 120 python tools/apply_probe.py --dtype f64 --only-cg --cg 100 2>&1 | tail -1
echo "== plain whole"; TCA_BAND_SCHED=whole timeout 120 python tools/apply_probe.py --dtype f64 --only-cg --cg 100 2>&1 | tail -1
echo "== f32 B1'"; TCA_B1=1 timeout 120 python tools/apply_probe.py --dtype f32 --only-cg --cg 100 2>&1 | tail -1
echo "== f32 unfused"; timeout 120 python tools/apply_probe.py --dtype f32 --only-cg --cg 100 2>&1 | tail -1
