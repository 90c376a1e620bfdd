"""bench.py's multi-GPU launcher, exercised on CPU (gloo, no GPU work):
`--gpus N` without a torchrun environment re-launches itself with N ranks,
and a torchrun environment whose WORLD_SIZE differs from --gpus is refused."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env(**kw):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT")}
    env.update(kw)
    return env


def test_gpus_2_starts_two_ranks():
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--mock"], capture_output=True, text=True,
                       timeout=300, env=_env(), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["max_ms"] == 2.0  # max over ranks of 1.0 + rank
    # [rank, local_rank, world, shard lo, shard hi]: one global batch of 8192 split in two (strong scaling)
    assert line["ranks"] == [[0, 0, 2, 0, 4096], [1, 1, 2, 4096, 8192]]


def test_world_size_must_match_gpus():
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--mock"], capture_output=True, text=True,
                       timeout=120, env=_env(RANK="0", LOCAL_RANK="0", WORLD_SIZE="1"), cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE=1 but --gpus 2" in (r.stderr + r.stdout)


def test_single_process_default():
    r = subprocess.run([sys.executable, BENCH, "--mock"], capture_output=True, text=True, timeout=120,
                       env=_env(), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["ranks"] == [[0, 0, 1, 0, 8192]]
