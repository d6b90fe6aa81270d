"""bench.py --gpus N starts its own ranks (one process per GPU) when it is not
already under torchrun, and every rank sees the same world. Checked on CPU
with gloo through the bench's own launcher path (--selftest-launch replaces
the GPU work with one all-reduce)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                          "--selftest-launch"], capture_output=True, text=True, timeout=240, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_two_ranks_spawned():
    r = _run(2)
    assert r["n_gpus"] == 2 and r["ranks_seen"] == 2


def test_single_rank_runs_inline():
    r = _run(1)
    assert r["n_gpus"] == 1 and r["ranks_seen"] == 1
