"""bench.py's driver contract on CPU: `--gpus N` without WORLD_SIZE re-executes itself as N ranks
(torch.distributed.run on 127.0.0.1) and rank 0 prints one JSON line with n_gpus = N (the
reference arm runs without a GPU); a WORLD_SIZE that disagrees with --gpus fails loudly."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, env=env, cwd=ROOT)


def test_gpus_n_spawns_n_ranks_and_prints_one_line():
    r = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "3", "--sample-seconds", "0.3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] == 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "2", "--impl", "reference", "--steps", "1"], env_extra={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)


def test_spawn_command_uses_loopback_rendezvous():
    sys.path.insert(0, ROOT)
    import bench
    cmd = bench.spawn_command(["--gpus", "8", "--steps", "5"], 8, 29501)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29501" in cmd
    assert cmd[-3:] == ["--gpus", "8", "--steps", "5"][-3:]
