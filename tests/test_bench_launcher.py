"""bench.py's multi-rank launcher on CPU (no GPU): `python bench.py --gpus 2` outside
torchrun must start 2 ranks itself (torch.distributed.run, 127.0.0.1), shard the
global batch and gather the outputs across ranks (gloo stand-in for NCCL), and
rank 0 must print one JSON line with n_gpus == 2; a WORLD_SIZE that disagrees with
--gpus is an error (VERDICT round 1 'make (e) measurable')."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env():
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["OMP_NUM_THREADS"] = "1"
    return env


def test_bench_gpus2_spawns_two_ranks():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--launcher-check", "--B", "8"], capture_output=True, text=True,
                       timeout=300, env=_env(), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["gpus_flag"] == 2
    assert line["per_rank_batch"] == 4 and line["gather_ok"] is True


def test_bench_world_size_mismatch_is_an_error():
    env = _env()
    env.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT="29999")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--launcher-check"], capture_output=True, text=True, timeout=120, env=env,
                       cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE=1 but --gpus 2" in (r.stderr + r.stdout)
