"""Run a few cfg2 solves of one solver (profiling driver for ncu).

    python tools/one_solve.py [--solver fista] [--dtype float64] [--reps 4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1007_3753_b200 import device as dv, synth
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig, StoppingRule
    ap = argparse.ArgumentParser()
    ap.add_argument("--solver", default="fista")
    ap.add_argument("--dtype", default="float64")
    ap.add_argument("--reps", type=int, default=4)
    args = ap.parse_args()
    P = synth.make_problem(synth.CFG2)
    D = dv.DeviceDictionary(P.A, dtype=args.dtype)
    Pd = ProblemInstance.__new__(ProblemInstance)
    Pd.A, Pd.b, Pd.ground_truth, Pd.noise_sigma = D, P.b, P.ground_truth, P.noise_sigma
    rel = StoppingRule("relative-estimate", 1e-6)
    cfg = SolverConfig(lam=None, tol=1e-6, stopping=rel, options={"dtype": args.dtype})
    lam = 1e-2 * float(np.max(np.abs(P.A.T @ P.b)))
    if args.solver == "fista":
        from paper_1007_3753_b200.shrinkage import fista_solve as fn
        run = lambda: fn(Pd, cfg)
    elif args.solver == "dalm":
        from paper_1007_3753_b200.alm import dalm_solve as fn
        run = lambda: fn(Pd, SolverConfig(tol=1e-6, stopping=rel, max_iter=300))
    elif args.solver == "palm":
        from paper_1007_3753_b200.alm import palm_solve as fn
        run = lambda: fn(Pd, cfg)
    elif args.solver == "gpsr":
        from paper_1007_3753_b200.gradient_projection import gpsr_solve as fn
        run = lambda: fn(Pd, lam, cfg)
    elif args.solver == "homotopy":
        from paper_1007_3753_b200.homotopy import homotopy_solve as fn
        run = lambda: fn(Pd, lam, SolverConfig())
    elif args.solver == "ist":
        from paper_1007_3753_b200.shrinkage import ist_solve as fn
        run = lambda: fn(Pd, None, cfg)
    elif args.solver == "tnipm":
        from paper_1007_3753_b200.gradient_projection import tnipm_solve as fn
        run = lambda: fn(Pd, lam, cfg)
    else:
        raise SystemExit("unknown solver")
    for _ in range(args.reps):
        r = run()
    torch.cuda.synchronize()
    print(args.solver, "iterations", r.iterations)


if __name__ == "__main__":
    main()
