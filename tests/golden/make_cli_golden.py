"""Golden fixtures for the CLI wire formats, made by running the REAL
reference CLI (ell1.cli.run) in the build container:

    cp -r /root/reference/pkg /tmp/ell1ref && (cd /tmp/ell1ref && python setup.py build_ext --inplace)
    PYTHONPATH=/tmp/ell1ref/src python tests/golden/make_cli_golden.py

Writes tests/golden/cli/: gen outputs (A.csv, b.csv, x0.csv), solve / cab
result JSONs, and manifest.json (argv and exit code of every run)."""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")

RUNS = [
    ("gen", ["gen", "--n", "60", "--d", "30", "--k", "4", "--seed", "3", "--noise-sigma", "0.001",
             "--matrix", "A.csv", "--rhs", "b.csv", "--truth", "x0.csv"]),
    ("solve_fista", ["solve", "--algo", "fista", "--matrix", "A.csv", "--rhs", "b.csv", "--seed", "3",
                     "--out", "solve_fista.json"]),
    ("solve_dalm", ["solve", "--algo", "dalm", "--matrix", "A.csv", "--rhs", "b.csv", "--max-iter", "300",
                    "--out", "solve_dalm.json"]),
    ("solve_homotopy", ["solve", "--algo", "homotopy", "--matrix", "A.csv", "--rhs", "b.csv",
                        "--lambda", "0.01", "--out", "solve_homotopy.json"]),
    ("solve_gp", ["solve", "--algo", "gp", "--matrix", "A.csv", "--rhs", "b.csv", "--out", "solve_gp.json"]),
    ("solve_budget", ["solve", "--algo", "fista", "--matrix", "A.csv", "--rhs", "b.csv", "--max-iter", "3",
                      "--out", "solve_budget.json"]),
    ("cab_homotopy", ["cab", "--algo", "homotopy", "--matrix", "A.csv", "--rhs", "b.csv",
                      "--out", "cab_homotopy.json"]),
    ("cab_dalm", ["cab", "--algo", "dalm", "--matrix", "A.csv", "--rhs", "b.csv", "--e-weight", "2",
                  "--max-iter", "2000", "--tol", "1e-6", "--out", "cab_dalm.json"]),
]


ALIGN_RUNS = [
    ("align_palm", ["align", "--algo", "palm", "--basis", "B.csv", "--rhs", "balign.csv",
                    "--out", "align_palm.json"]),
    ("align_ist", ["align", "--algo", "ist", "--basis", "B.csv", "--rhs", "balign.csv", "--lambda", "0.05",
                   "--tol", "1e-7", "--max-iter", "20000", "--out", "align_ist.json"]),
    ("align_homotopy", ["align", "--algo", "homotopy", "--basis", "B.csv", "--rhs", "balign.csv",
                        "--out", "align_homotopy.json"]),
    ("align_gp", ["align", "--algo", "gp", "--basis", "B.csv", "--rhs", "balign.csv", "--max-iter", "200",
                  "--out", "align_gp.json"]),
]


def main():
    from ell1 import cli
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from tests.golden.align_cases import align_instance
    import numpy as np
    os.makedirs(OUT, exist_ok=True)
    B, b = align_instance(seed=21, d=90, m=6)
    np.savetxt(os.path.join(OUT, "B.csv"), B, fmt="%.17g", delimiter=",")
    np.savetxt(os.path.join(OUT, "balign.csv"), b[:, None], fmt="%.17g", delimiter=",")
    os.environ["ELL1_OUT_DIR"] = OUT
    manifest = []
    for name, argv in RUNS + ALIGN_RUNS:
        # inputs are read relative to the fixture directory
        argv = [os.path.join(OUT, a) if a.endswith(".csv") and name != "gen" else a for a in argv]
        rc = cli.run(argv)
        manifest.append({"name": name, "argv": [os.path.basename(a) if a.endswith(".csv") else a
                                                for a in argv], "exit": rc})
        print(name, rc)
    with open(os.path.join(OUT, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
        fh.write("\n")


if __name__ == "__main__":
    sys.exit(main())
