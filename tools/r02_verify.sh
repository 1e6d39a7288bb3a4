mkdir -p gpurun_out/r02g
python tools/apply_probe.py --dtype f64 --reps 30 --cg 30 > gpurun_out/r02g/probe.log 2>&1
python tools/apply_probe.py --dtype f32 --reps 30 --cg 30 >> gpurun_out/r02g/probe.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02g/gputest.log 2>&1
python bench.py > gpurun_out/r02g/bench_f64.log 2>&1
python bench.py --dtype f32 --cfg4-iters 0 > gpurun_out/r02g/bench_f32.log 2>&1
tail -3 gpurun_out/r02g/gputest.log
cat gpurun_out/r02g/probe.log | tail -20
