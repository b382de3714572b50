"""bench.py's multi-rank plumbing on the CPU: `--dry-run --gpus 2` spawns two ranks over gloo
(rendezvous on 127.0.0.1), runs the expert-parallel exchange and timing code paths and prints the
driver's one JSON line with n_gpus == 2 (a driver `--gpus N` run must report N)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_bench_dry_run_two_ranks():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29561")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--dry-run", "--gpus", "2", "--steps", "3",
                          "--warmup", "3"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True
    assert d["steps"] == 3 and d["warmup"] == 3
    for key in ("metric", "unit", "ms_per_step", "higher_is_better", "scaling"):
        assert key in d
    assert d["ms_per_step"] > 0
