"""Golden fixtures for the alignment solvers, made by
running the REAL reference (ell1.robust.align_*_solve) in the build container:

    PYTHONPATH=/tmp/ell1ref/src python tests/golden/make_align_golden.py

Inputs come from align_instance() (tests/golden/align_cases.py, seeded);
outputs go to tests/golden/align_golden.npz."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests.golden.align_cases import CASES, align_instance  # noqa: E402


def main():
    from ell1.model import SolverConfig
    from ell1.robust import (AlignmentProblem, align_gp_solve, align_homotopy_solve, align_ist_solve,
                             align_palm_solve)
    out = {}
    for name, c in CASES.items():
        B, b = align_instance(**c["recipe"])
        prob = AlignmentProblem(B, b)
        cfg = SolverConfig(tol=c["tol"], max_iter=c["max_iter"], options=c.get("options", {}),
                           lam=c.get("lam") if c["solver"] == "homotopy" else None)
        if c["solver"] == "palm":
            w, e = align_palm_solve(prob, cfg)
        elif c["solver"] == "homotopy":
            w, e = align_homotopy_solve(prob, cfg)
        elif c["solver"] == "gp":
            w, e = align_gp_solve(prob, c.get("lam"), cfg)
        else:
            w, e = align_ist_solve(prob, c.get("lam"), cfg)
        out[name + "_w"] = w
        out[name + "_e"] = e
        print(name, np.linalg.norm(e, 1))
    np.savez_compressed(os.path.join(HERE, "align_golden.npz"), **out)


if __name__ == "__main__":
    main()
