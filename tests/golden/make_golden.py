"""Generate the golden parity fixtures by running the REAL reference.

Run in the build container only (the reference is not on the GPU box):

    cp -r /root/reference/pkg /tmp/ell1ref
    (cd /tmp/ell1ref && python setup.py build_ext --inplace)   # compiled _accel
    PYTHONPATH=/tmp/ell1ref/src:. python tests/golden/make_golden.py [--sizes small,cfg1,...]

Each case (tests/golden/cases.py) is rebuilt from its seed recipe, solved
with the reference's public entry point, and stored as tests/golden/<id>.npz
(x_star, iterations, converged, trace[N,4], notes, plus e for CAB cases).
"""

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests.golden.cases import CASES, build_inputs, resolve_lambda  # noqa: E402


def run_reference(case):
    import ell1
    from ell1 import alm, gradient_projection, homotopy, pdipa, robust, shrinkage
    from ell1.model import ProblemInstance, SolverConfig, StoppingRule

    assert ell1.kernels_compiled, "build the reference's _accel first"
    A, b, gt = build_inputs(case["recipe"])
    cfg = dict(case["cfg"])
    lam = resolve_lambda(cfg, A, b)
    stop = cfg.get("stopping")
    config = SolverConfig(lam=lam, tol=cfg.get("tol", 1e-6),
                          max_iter=cfg.get("max_iter", 5000),
                          stopping=StoppingRule(*stop) if stop else None,
                          options=dict(cfg.get("options", {})))
    solver = case["solver"]
    extra = {}
    if solver.startswith("cab:"):
        x, e, res = robust.cab_solve(A, b, solver[4:], config)
        extra["e"] = e
        extra["w"] = res.x_star
    else:
        P = ProblemInstance(A, b, ground_truth=gt)
        if solver == "fista":
            res = shrinkage.fista_solve(P, config)
        elif solver == "ist":
            sched = None
            if case["extra"].get("schedule") == "flat":
                sched = shrinkage.ContinuationSchedule(lam, 0.5, lam)
            res = shrinkage.ist_solve(P, sched, config)
        elif solver == "palm":
            res = alm.palm_solve(P, config)
        elif solver == "dalm":
            res = alm.dalm_solve(P, config)
        elif solver == "gpsr":
            res = gradient_projection.gpsr_solve(P, lam, config)
        elif solver == "tnipm":
            res = gradient_projection.tnipm_solve(P, lam, config)
        elif solver == "homotopy":
            target = lam if lam is not None else config.resolved_lambda(P)
            extra["target"] = target
            res = homotopy.homotopy_solve(P, target, config)
        elif solver == "pdipa":
            res = pdipa.pdipa_solve(P, config)
        else:
            raise ValueError(solver)
        x = res.x_star
    trace = np.array([tuple(t) for t in res.trace], dtype=np.float64).reshape(-1, 4)
    return dict(x=np.asarray(x, dtype=np.float64), iterations=res.iterations,
                converged=res.converged, trace=trace,
                notes=json.dumps(list(res.notes)),
                wall=res.wall_time_seconds, **extra)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="small,cfg1,cfg2,cfg5")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    sizes = set(args.sizes.split(","))
    for case in CASES:
        if case["size"] not in sizes:
            continue
        if args.only and case["id"] != args.only:
            continue
        t0 = time.perf_counter()
        out = run_reference(case)
        np.savez_compressed(os.path.join(HERE, case["id"] + ".npz"), **out)
        print("%-24s it=%-5d conv=%-5s %.2fs" % (case["id"], out["iterations"],
                                                 out["converged"], time.perf_counter() - t0))


if __name__ == "__main__":
    main()
