# deferred-x (MODE 2, extra streaming warp) A/B on config 3: CG us/iteration and apply time in CG
for v in 1 0; do TCA_DX=$v python tools/cg_probe.py --dtype f32; done
TCA_DX=1 python tools/cg_probe.py --dtype f32 --solver pcg --iters 100; TCA_DX=0 python tools/cg_probe.py --dtype f32 --solver pcg --iters 100
python tools/cg_probe.py --dtype f64
