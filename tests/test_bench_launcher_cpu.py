"""bench.py's multi-rank launcher on CPU: `python bench.py --gpus N` without
WORLD_SIZE re-runs itself under torch.distributed.run (one process per GPU,
rendezvous on 127.0.0.1).  Here the same launcher starts two gloo ranks of a
small script that all-reduces a value, takes the max over ranks like the bench
does, and prints one JSON line from rank 0 only."""
import json
import os
import subprocess
import sys
import textwrap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RANK_SCRIPT = textwrap.dedent("""
    import json, os, sys, torch, torch.distributed as dist
    dist.init_process_group("gloo")
    r, w = dist.get_rank(), dist.get_world_size()
    assert w == int(os.environ["WORLD_SIZE"]) and os.environ["MASTER_ADDR"] == "127.0.0.1"
    t = torch.tensor([float(r + 1)])
    dist.all_reduce(t)
    m = torch.tensor([10.0 * (r + 1)])
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    if r == 0:
        print(json.dumps({"n_gpus": w, "sum": t.item(), "max": m.item(), "args": sys.argv[1:]}), flush=True)
    dist.destroy_process_group()
""")


def test_spawn_ranks_two_gloo_processes_one_line(tmp_path):
    script = tmp_path / "rank.py"
    script.write_text(RANK_SCRIPT)
    code = ("import sys; sys.path.insert(0, %r); import bench; "
            "sys.exit(bench.spawn_ranks(2, %r, ['--steps', '3']))" % (ROOT, str(script)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OMP_NUM_THREADS"] = "1"
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    out = json.loads(lines[0])
    assert out == {"n_gpus": 2, "sum": 3.0, "max": 20.0, "args": ["--steps", "3"]}


def test_bench_gpus_flag_without_devices_fails_loudly():
    """--gpus 2 on a host without two CUDA devices: a clear error, not a silent
    one-GPU run reported as two."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "visible CUDA device" in r.stderr
