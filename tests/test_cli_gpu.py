"""CLI solves on the GPU against the reference CLI's own outputs on the same
instance (tests/golden/cli, made by make_cli_golden.py): same exit code,
same JSON keys in the same order, same iteration count and convergence flag,
x within the north-star parity tolerance (wall time is not compared)."""

import json
import os
import shutil

import numpy as np
import pytest

from paper_1007_3753_b200 import cli

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")

with open(os.path.join(GOLD, "manifest.json")) as _fh:
    RUNS = [m for m in json.load(_fh) if m["name"] != "gen"]


@pytest.mark.parametrize("run", RUNS, ids=[m["name"] for m in RUNS])
def test_cli_run_matches_reference(tmp_path, monkeypatch, run):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    monkeypatch.delenv("ELL1_OUT_DIR", raising=False)
    monkeypatch.chdir(tmp_path)
    for name in os.listdir(GOLD):
        if name.endswith(".csv"):
            shutil.copy(os.path.join(GOLD, name), name)
    argv = list(run["argv"])
    out = argv[argv.index("--out") + 1]
    assert cli.run(argv) == run["exit"]
    with open(out) as fh:
        ours = json.load(fh)
    with open(os.path.join(GOLD, out)) as fh:
        ref = json.load(fh)
    assert list(ours.keys()) == list(ref.keys())
    assert ours["config_echo"] == ref["config_echo"]
    for key in ("algo", "n", "d", "iterations", "converged", "seed"):
        assert ours[key] == ref[key], key
    if ref["lambda"] is None:
        assert ours["lambda"] is None
    else:
        assert ours["lambda"] == pytest.approx(ref["lambda"], rel=1e-12)
    x, xr = np.array(ours["x"]), np.array(ref["x"])
    assert np.linalg.norm(x - xr) <= 1e-6 * max(np.linalg.norm(xr), 1e-300)
    if "e" in ref:
        e, er = np.array(ours["e"]), np.array(ref["e"])
        assert np.linalg.norm(e - er) <= 1e-6 * max(np.linalg.norm(er), 1e-300)
    assert ours["objective"] == pytest.approx(ref["objective"], rel=1e-9, abs=1e-12)
