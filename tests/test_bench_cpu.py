"""bench.py's launcher on CPU: ``--gpus 2`` outside torchrun re-launches
itself under torch.distributed.run, the ranks rendezvous over gloo on
127.0.0.1 and drive the sharded one-allreduce-per-round protocol; rank 0
prints one JSON line with n_gpus = 2 (dry run: no timing claim)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run"] + list(args),
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_dry_run_two_ranks():
    out = _run("--gpus", "2")
    assert out["n_gpus"] == 2 and out["backend"] == "gloo"
    assert out["converged"] and out["iterations"] > 0


def test_dry_run_single():
    out = _run()
    assert out["n_gpus"] == 1
