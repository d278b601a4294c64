"""CLI front end (paper_1007_3753_b200.cli) without a GPU: the reference's
test_cli scenarios that do not solve — generator output byte-identical to
the reference CLI's (tests/golden/cli, made by make_cli_golden.py), "%.17g"
round trips, usage errors -> exit 2 with a diagnostic, unsupported
subcommands exit 2."""

import json
import os
import shutil

import numpy as np
import pytest

from paper_1007_3753_b200 import cli

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


@pytest.fixture
def workdir(tmp_path, monkeypatch):
    monkeypatch.delenv("ELL1_OUT_DIR", raising=False)
    monkeypatch.chdir(tmp_path)
    return tmp_path


def _manifest():
    with open(os.path.join(GOLD, "manifest.json")) as fh:
        return {m["name"]: m for m in json.load(fh)}


def test_gen_byte_identical_to_reference(workdir):
    argv = _manifest()["gen"]["argv"]
    assert cli.run(argv) == 0
    for name in ("A.csv", "b.csv", "x0.csv"):
        with open(name, "rb") as a, open(os.path.join(GOLD, name), "rb") as b:
            assert a.read() == b.read(), name


def test_gen_deterministic_and_seed_sensitive(workdir):
    base = ["gen", "--n", "20", "--d", "10", "--k", "3", "--rhs", "b.csv"]
    assert cli.run(base + ["--seed", "1", "--matrix", "A1.csv"]) == 0
    assert cli.run(base + ["--seed", "1", "--matrix", "A2.csv"]) == 0
    assert cli.run(base + ["--seed", "2", "--matrix", "A3.csv"]) == 0
    one, two, three = (open(p, "rb").read() for p in ("A1.csv", "A2.csv", "A3.csv"))
    assert one == two and one != three


def test_round_trip_bit_identical(workdir):
    assert cli.run(["gen", "--n", "30", "--d", "12", "--k", "4", "--seed", "5", "--noise-sigma", "0.1",
                    "--matrix", "A.csv", "--rhs", "b.csv", "--truth", "x.csv"]) == 0
    from paper_1007_3753_b200 import synth
    P = synth.make_instance(synth.GenSpec(n=30, d=12, k=4, seed=5, noise_sigma=0.1))
    assert np.array_equal(np.loadtxt("A.csv", delimiter=",", ndmin=2), P.A)
    assert np.array_equal(np.loadtxt("b.csv", delimiter=","), P.b)
    assert np.array_equal(np.loadtxt("x.csv", delimiter=","), P.ground_truth)


def test_outputs_land_in_env_dir(workdir, monkeypatch):
    out = workdir / "outdir"
    out.mkdir()
    monkeypatch.setenv("ELL1_OUT_DIR", str(out))
    assert cli.run(["gen", "--n", "8", "--d", "4", "--k", "2", "--matrix", "A.csv", "--rhs", "b.csv"]) == 0
    assert (out / "A.csv").exists() and (out / "b.csv").exists()


def test_gen_validation_exit_2(workdir, capsys):
    assert cli.run(["gen", "--n", "5", "--d", "4", "--k", "9", "--matrix", "A.csv", "--rhs", "b.csv"]) == 2
    assert "error" in capsys.readouterr().err


@pytest.mark.parametrize("argv", [
    ["solve", "--matrix", "missing.csv", "--rhs", "b.csv", "--out", "r.json"],
    ["solve", "--matrix", "bad.csv", "--rhs", "b.csv", "--out", "r.json"],
    ["solve", "--matrix", "A.csv", "--rhs", "two.csv", "--out", "r.json"],
    ["solve", "--matrix", "A.csv", "--rhs", "short.csv", "--out", "r.json"],
    ["solve", "--bogus-flag", "--matrix", "A.csv", "--rhs", "b.csv", "--out", "r.json"],
    ["solve", "--algo", "nope", "--matrix", "A.csv", "--rhs", "b.csv", "--out", "r.json"],
    ["cab", "--matrix", "A.csv", "--rhs", "short.csv", "--out", "r.json"],
    ["phase", "--algo", "fista", "--n", "20", "--grid", "4by4", "--out", "g.csv"],
    ["phase", "--algo", "fista", "--n", "20", "--grid", "2x2", "--out", "g.csv", "--svg", "g.svg"],
    ["noise-sweep", "--mode", "vary-d", "--solvers", "fista", "--n", "20", "--out", "s.csv"],
    ["noise-sweep", "--mode", "vary-k", "--solvers", "nope", "--n", "20", "--d", "10",
     "--rho-values", "0.1", "--out", "s.csv"],
    ["align", "--basis", "B.csv", "--rhs", "b.csv", "--out", "r.json"],
    ["report", "--input", "g.csv", "--svg", "g.svg"],
])
def test_usage_errors_exit_2(workdir, argv, capsys):
    shutil.copy(os.path.join(GOLD, "A.csv"), "A.csv")
    shutil.copy(os.path.join(GOLD, "b.csv"), "b.csv")
    with open("bad.csv", "w") as fh:
        fh.write("1,2\n3,x\n")
    with open("two.csv", "w") as fh:
        fh.write("1,2\n3,4\n")
    with open("short.csv", "w") as fh:
        fh.write("1\n2\n")
    assert cli.run(argv) == 2
    err = capsys.readouterr().err
    assert err.strip(), "a diagnostic on stderr"


def test_dimension_mismatch_names_both(workdir, capsys):
    shutil.copy(os.path.join(GOLD, "A.csv"), "A.csv")
    with open("short.csv", "w") as fh:
        fh.write("1\n2\n")
    assert cli.run(["solve", "--matrix", "A.csv", "--rhs", "short.csv", "--out", "r.json"]) == 2
    err = capsys.readouterr().err
    assert "matrix" in err and "rhs" in err


def test_result_payload_key_order_matches_reference():
    with open(os.path.join(GOLD, "solve_fista.json")) as fh:
        ref_keys = list(json.load(fh).keys())
    from paper_1007_3753_b200.model import SolverConfig
    ours = cli.result_payload("fista", 60, 30, 0.1, 5, True, 0.0, np.zeros(3), 1.0, 0.0,
                              SolverConfig(), 3)
    assert list(ours.keys()) == ref_keys
    with open(os.path.join(GOLD, "cab_dalm.json")) as fh:
        ref = json.load(fh)
    ours = cli.result_payload("dalm", 60, 30, None, 5, True, 0.0, np.zeros(3), 1.0, 0.0,
                              SolverConfig(tol=1e-6, max_iter=2000, options={"e_weight": 2.0}), None,
                              e=np.zeros(2))
    assert list(ours.keys()) == list(ref.keys())
    assert list(ours["config_echo"].keys()) == list(ref["config_echo"].keys())


def test_alignment_problem_validation():
    from paper_1007_3753_b200.robust import AlignmentProblem
    with pytest.raises(ValueError):
        AlignmentProblem(np.ones((3, 5)), np.ones(3))      # wide
    with pytest.raises(ValueError):
        AlignmentProblem(np.ones((6, 2)), np.ones(5))      # length mismatch
    p = AlignmentProblem(np.ones((6, 2)), np.ones(6))
    assert (p.d, p.m) == (6, 2)
