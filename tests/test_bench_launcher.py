"""bench.py --gpus N spawns N ranks itself when no torchrun environment is
set (the driver may call it either way); each rank gets its own angular
shard.  Checked with --dry-run under gloo (no GPU work)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_two_ranks_two_shards():
    line = run_bench("--gpus", "2", "--dry-run")
    assert line["n_gpus"] == 2
    assert [r["rank"] for r in line["ranks"]] == [0, 1]
    assert [tuple(r["shard"]) for r in line["ranks"]] == [(0, 2), (1, 2)]


def test_one_gpu_is_unsharded():
    line = run_bench("--dry-run")
    assert line["n_gpus"] == 1 and line["ranks"][0]["shard"] is None
