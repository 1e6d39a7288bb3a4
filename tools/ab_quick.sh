# quick apply A/B on config 3: tools/ab_quick.sh (uses the in-tree library)
for i in 1 2; do python tools/apply_probe.py --dtype f64 --reps 30 --cg 30; python tools/apply_probe.py --dtype f32 --reps 30 --cg 30; done
