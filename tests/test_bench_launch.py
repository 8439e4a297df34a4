"""bench.py launch contract on CPU: `bench.py --gpus N` outside torchrun
spawns N ranks itself (torch.distributed.run on 127.0.0.1), every rank joins
the process group, and stdout carries exactly one JSON line from rank 0.
--dry-run swaps the GPU work for a gloo all_reduce of the ranks."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus", [2, 3])
def test_bench_gpus_flag_spawns_ranks(gpus):
    out = _run("--gpus", str(gpus), "--dry-run")
    assert out["n_gpus"] == gpus and out["ranks"] == gpus
    assert out["rank_sum"] == gpus * (gpus - 1) // 2


def test_bench_single_gpu_stays_in_process():
    out = _run("--dry-run")
    assert out["n_gpus"] == 1 and out["ranks"] == 1
