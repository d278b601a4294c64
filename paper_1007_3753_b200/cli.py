"""Command-line front end on the B200 backend.

Mirrors the reference's `ell1` CLI (cli.py) — subcommands, flags, file
formats and exit codes — with every solve running on the device:

* wire formats (cli.py:1-9, 54-83): plain CSV, UTF-8, LF, one matrix row per
  line, "%.17g" numbers, no header, vectors single-column; result JSON with
  the reference's fixed key order (cli.py:116-135), 2-space indent, trailing
  newline; relative output paths resolved against $ELL1_OUT_DIR.
* exit codes: 0 success, 1 solver did not meet its convergence test
  (results still written) or broke down numerically, 2 usage error.

Subcommands: solve, gen, cab, phase, noise-sweep, align (cli.py:137-350).
SVG rendering (`report`, --svg) is not part of this backend and exits 2
with a diagnostic.

    python -m paper_1007_3753_b200.cli solve --algo fista --matrix A.csv --rhs b.csv --out r.json
"""

import argparse
import json
import os
import re
import sys

import numpy as np

from paper_1007_3753_b200 import harness, synth
from paper_1007_3753_b200.exceptions import DeviceError, NumericalError
from paper_1007_3753_b200.model import (ProblemInstance, SolverConfig, kkt_from_correlation,
                                        kkt_residual, objective)
from paper_1007_3753_b200.solvers import SOLVER_NAMES, solve_named

FMT = "%.17g"
EQUALITY_ALGOS = ("pdipa", "palm", "dalm")            # no penalty weight (cli.py:37)
CAB_ALGOS = ("pdipa", "homotopy", "gp", "ist", "fista", "palm", "dalm")


class UsageError(Exception):
    """Reported on stderr with exit code 2."""


# ------------------------------------------------------------------ file I/O
def out_path(path):
    base = os.environ.get("ELL1_OUT_DIR")
    return os.path.join(base, path) if base and not os.path.isabs(path) else path


def read_csv(path, what):
    try:
        return np.loadtxt(path, delimiter=",", dtype=np.float64, ndmin=2)
    except OSError as exc:
        raise UsageError("cannot read %s file %r: %s" % (what, path, exc))
    except ValueError as exc:
        raise UsageError("malformed CSV in %s file %r: %s" % (what, path, exc))


def read_vector(path, what):
    arr = read_csv(path, what)
    if arr.shape[1] != 1:
        raise UsageError("%s file %r must be a single-column CSV, got %d columns"
                         % (what, path, arr.shape[1]))
    return arr[:, 0].copy()


def write_matrix(path, M):
    np.savetxt(out_path(path), np.atleast_2d(M), fmt=FMT, delimiter=",")


def write_vector(path, v):
    np.savetxt(out_path(path), np.asarray(v)[:, None], fmt=FMT, delimiter=",")


def write_json(path, payload):
    with open(out_path(path), "w", encoding="utf-8", newline="\n") as fh:
        json.dump(payload, fh, indent=2)
        fh.write("\n")


def same_rows(name_a, shape, name_b, length):
    if shape[0] != length:
        raise UsageError("%s is %dx%d but %s has length %d" % (name_a, shape[0], shape[1], name_b, length))


# ------------------------------------------------------------------ payloads
def make_config(args, tol, max_iter):
    options = {}
    if getattr(args, "e_weight", None) is not None:
        options["e_weight"] = args.e_weight
    return SolverConfig(lam=getattr(args, "lam", None),
                        tol=tol if args.tol is None else args.tol,
                        max_iter=max_iter if args.max_iter is None else args.max_iter,
                        options=options)


def config_echo(cfg):
    echo = {"tol": cfg.tol, "max_iter": cfg.max_iter, "lam": cfg.lam}
    for key in sorted(cfg.options):
        echo[key] = cfg.options[key]
    return echo


def result_payload(algo, n, d, lam, iterations, converged, wall, x, obj, kkt, cfg, seed, e=None):
    """Key order of the reference's result JSON (cli.py:116-135)."""
    out = {"algo": algo, "n": n, "d": d, "lambda": lam, "iterations": iterations,
           "converged": converged, "wall_time_seconds": wall, "x": [float(v) for v in x]}
    if e is not None:
        out["e"] = [float(v) for v in e]
    out["objective"] = obj
    out["kkt_residual"] = kkt
    out["config_echo"] = config_echo(cfg)
    out["seed"] = seed
    return out


# ------------------------------------------------------------------ commands
def cmd_solve(args):
    """cli.py:137-163: one named solver on a CSV instance."""
    A = read_csv(args.matrix, "matrix")
    b = read_vector(args.rhs, "rhs")
    same_rows("matrix", A.shape, "rhs", b.size)
    P = ProblemInstance(A, b)
    cfg = make_config(args, 1e-6, 5000)
    res = solve_named(args.algo, P, cfg)
    x = res.x_star
    lam = None if args.algo in EQUALITY_ALGOS else cfg.resolved_lambda(P)
    if not lam:
        # equality form (or homotopy to a zero target): l1 norm + constraint violation
        obj = float(np.abs(x).sum())
        kkt = float(np.abs(A @ x - b).max())
    else:
        obj = objective(x, P, lam)
        kkt = kkt_residual(x, P, lam)
    write_json(args.out, result_payload(args.algo, P.n, P.d, lam, res.iterations, bool(res.converged),
                                        res.wall_time_seconds, x, obj, kkt, cfg, args.seed))
    return 0 if res.converged else 1


def cmd_gen(args):
    """cli.py:166-177: a synthetic instance as CSV (host generator, reference recipe)."""
    try:
        spec = synth.GenSpec(n=args.n, d=args.d, k=args.k, seed=args.seed, noise_sigma=args.noise_sigma)
    except ValueError as exc:
        raise UsageError(str(exc))
    P = synth.make_instance(spec)
    write_matrix(args.matrix, P.A)
    write_vector(args.rhs, P.b)
    if args.truth is not None:
        write_vector(args.truth, P.ground_truth)
    return 0


def cmd_cab(args):
    """cli.py:265-295: sparse signal + sparse corruption on [A, I/e_weight]."""
    from paper_1007_3753_b200.robust import cab_solve
    A = read_csv(args.matrix, "matrix")
    b = read_vector(args.rhs, "rhs")
    same_rows("matrix", A.shape, "rhs", b.size)
    cfg = make_config(args, 1e-8, 4000)
    x, e, res = cab_solve(A, b, args.algo, cfg)
    d, n = A.shape
    ew = cfg.opt("e_weight", 1.0)
    w = np.concatenate([x, e * ew])                      # coefficients on [A, I / e_weight]
    r = b - (A @ w[:n] + w[n:] / ew)
    if args.algo in EQUALITY_ALGOS:
        lam = None
        obj = float(np.abs(w).sum())
        kkt = float(np.abs(r).max())
    else:
        c = np.concatenate([A.T @ r, r / ew])
        lam = cfg.lam
        if lam is None:                      # the default the backend resolved on [A, I/e_weight]
            lam = 1e-2 * float(np.abs(np.concatenate([A.T @ b, b / ew])).max())
        obj = 0.5 * float(r @ r) + lam * float(np.abs(w).sum())
        kkt = kkt_from_correlation(w, c, lam)
    write_json(args.out, result_payload(args.algo, n, d, lam, res.iterations, bool(res.converged),
                                        res.wall_time_seconds, x, obj, kkt, cfg, args.seed, e=e))
    return 0 if res.converged else 1


def parse_grid(text):
    m = re.fullmatch(r"(\d+)x(\d+)", text)
    if not m or int(m.group(1)) < 1 or int(m.group(2)) < 1:
        raise UsageError("grid must look like 16x16 (rho cells x delta cells), got %r" % text)
    R, Cn = int(m.group(1)), int(m.group(2))
    # interior points of (0, 1) on both axes (cli.py:180-188)
    return tuple((i + 1) / (R + 1) for i in range(R)), tuple((j + 1) / (Cn + 1) for j in range(Cn))


def no_svg(args):
    if getattr(args, "svg", None) is not None:
        raise UsageError("SVG rendering is not part of the B200 backend; render the CSV with "
                         "the reference's `ell1 report`")


def cmd_phase(args):
    """cli.py:202-223: success-rate grid on group launches (one dictionary per trial)."""
    no_svg(args)
    rho, delta = parse_grid(args.grid)
    cfg = make_config(args, 1e-8, 20000)
    grid = harness.run_phase_grid(args.algo, args.n, rho, delta, trials=args.trials,
                                  success_tol=args.success_tol, base_seed=args.seed, config=cfg,
                                  jobs=args.jobs)
    harness.phase_grid_to_csv(grid, out_path(args.out))
    if args.summary is not None:
        harness.write_summary_json(
            out_path(args.summary), "phase",
            {"algo": args.algo, "n": args.n, "grid": args.grid, "trials": args.trials,
             "seed": args.seed, "success_tol": args.success_tol},
            results={"cells": len(rho) * len(delta),
                     "mean_success_rate": float(grid.success_rate.mean())})
    return 0


def float_list(text, flag):
    try:
        vals = [float(t) for t in text.split(",") if t]
    except ValueError:
        raise UsageError("%s must be a comma-separated number list, got %r" % (flag, text))
    if not vals:
        raise UsageError("%s must not be empty" % flag)
    return vals


def cmd_noise_sweep(args):
    """cli.py:226-262."""
    no_svg(args)
    solvers = tuple(t for t in args.solvers.split(",") if t)
    if not solvers:
        raise UsageError("need at least one solver name")
    for name in solvers:
        if name != "gp" and name not in SOLVER_NAMES:
            raise UsageError("unknown solver %r (choose from %s)" % (name, ", ".join(SOLVER_NAMES)))
    if args.mode == "vary-d":
        if args.k is None or args.d_values is None:
            raise UsageError("vary-d needs --k and --d-values")
        spec = {"n": args.n, "k": args.k,
                "d_values": [int(v) for v in float_list(args.d_values, "--d-values")]}
    else:
        if args.d is None or args.rho_values is None:
            raise UsageError("vary-k needs --d and --rho-values")
        spec = {"n": args.n, "d": args.d, "rho_values": float_list(args.rho_values, "--rho-values")}
    spec["noise_sigma"] = args.noise_sigma
    cfg = make_config(args, 1e-6, 5000)
    sweep = harness.run_noise_sweep(solvers, args.mode, spec, trials=args.trials, base_seed=args.seed,
                                    config=cfg, jobs=args.jobs)
    harness.sweep_to_csv(sweep, out_path(args.out))
    if args.summary is not None:
        harness.write_summary_json(
            out_path(args.summary), "noise-sweep",
            {"mode": args.mode, "solvers": list(solvers), "trials": args.trials, "seed": args.seed,
             "noise_sigma": args.noise_sigma, "spec": {k: spec[k] for k in sorted(spec)}},
            results={"axis": list(sweep.axis_values)})
    return 0


def cmd_align(args):
    """cli.py:298-350: tall regression with sparse gross errors (PALM / IST on
    the device; iteration counts are not part of the alignment contract, so
    convergence is certified after the fact as in the reference)."""
    from paper_1007_3753_b200.robust import (AlignmentProblem, align_gp_solve, align_homotopy_solve,
                                             align_ist_solve, align_palm_solve)
    import time
    B = read_csv(args.basis, "basis")
    b = read_vector(args.rhs, "rhs")
    same_rows("basis", B.shape, "rhs", b.size)
    try:
        prob = AlignmentProblem(B, b)
    except ValueError as exc:
        raise UsageError(str(exc))
    cfg = make_config(args, 1e-8, 5000)
    t0 = time.perf_counter()
    if args.algo == "palm":
        w, e = align_palm_solve(prob, cfg)
    elif args.algo == "homotopy":
        w, e = align_homotopy_solve(prob, cfg)
    elif args.algo == "gp":
        w, e = align_gp_solve(prob, args.lam, cfg)
    else:
        w, e = align_ist_solve(prob, args.lam, cfg)
    wall = time.perf_counter() - t0
    r = b - B @ w - e
    if args.algo == "palm":
        lam = None
        obj = float(np.abs(e).sum())
        kkt = float(np.abs(r).max())
        converged = bool(np.linalg.norm(r) <= 10.0 * cfg.tol * max(1.0, np.linalg.norm(b)))
    else:
        lam = cfg.lam
        if lam is None:                      # 1e-2 x the peak least-squares residual (robust.py:270-273)
            w0 = np.linalg.solve(B.T @ B, B.T @ b)
            lam = 1e-2 * float(np.abs(b - B @ w0).max())
        obj = 0.5 * float(r @ r) + lam * float(np.abs(e).sum())
        grad_w = float(np.abs(B.T @ r).max())
        ke = kkt_from_correlation(e, r, lam)
        kkt = max(grad_w, ke)
        scale = max(1.0, float(np.abs(B.T @ b).max()))
        converged = bool(grad_w <= 10.0 * cfg.tol * scale and ke <= 10.0 * cfg.tol * lam)
    write_json(args.out, result_payload(args.algo, prob.m, prob.d, lam, None, converged, wall, w, obj, kkt,
                                        cfg, args.seed, e=e))
    return 0 if converged else 1


def cmd_unsupported(args):
    raise UsageError("`%s` is not provided by the B200 backend (%s)" % (
        args.subcommand, {"report": "SVG rendering"}[args.subcommand]))


# ------------------------------------------------------------------ parser
def _config_flags(p, with_lambda=True):
    if with_lambda:
        p.add_argument("--lambda", dest="lam", type=float, default=None)
    p.add_argument("--tol", type=float, default=None)
    p.add_argument("--max-iter", type=int, default=None)


def build_parser():
    algos = SOLVER_NAMES + ("gp",)
    top = argparse.ArgumentParser(prog="ell1", description="l1 solvers on the B200 (CSV/JSON I/O).")
    sub = top.add_subparsers(dest="subcommand", required=True)

    p = sub.add_parser("solve")
    p.add_argument("--algo", choices=algos, default="fista")
    p.add_argument("--matrix", required=True)
    p.add_argument("--rhs", required=True)
    _config_flags(p)
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_solve)

    p = sub.add_parser("gen")
    for flag in ("--n", "--d", "--k"):
        p.add_argument(flag, type=int, required=True)
    p.add_argument("--noise-sigma", type=float, default=0.0)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--matrix", required=True)
    p.add_argument("--rhs", required=True)
    p.add_argument("--truth", default=None)
    p.set_defaults(func=cmd_gen)

    p = sub.add_parser("phase")
    p.add_argument("--algo", choices=algos, required=True)
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--grid", required=True)
    p.add_argument("--trials", type=int, default=20)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--success-tol", type=float, default=1e-3)
    _config_flags(p)
    p.add_argument("--jobs", type=int, default=1)
    p.add_argument("--out", required=True)
    for flag, default in (("--svg", None), ("--levels", "50,90"), ("--title", None), ("--summary", None)):
        p.add_argument(flag, default=default)
    p.set_defaults(func=cmd_phase)

    p = sub.add_parser("noise-sweep")
    p.add_argument("--mode", choices=("vary-d", "vary-k"), required=True)
    p.add_argument("--solvers", required=True)
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--d-values", default=None)
    p.add_argument("--d", type=int, default=None)
    p.add_argument("--rho-values", default=None)
    p.add_argument("--noise-sigma", type=float, default=0.1)
    p.add_argument("--trials", type=int, default=10)
    p.add_argument("--seed", type=int, default=0)
    _config_flags(p)
    p.add_argument("--jobs", type=int, default=1)
    p.add_argument("--out", required=True)
    for flag, default in (("--svg", None), ("--metric", "mean_rel_error"), ("--title", None),
                          ("--summary", None)):
        p.add_argument(flag, default=default)
    p.set_defaults(func=cmd_noise_sweep)

    p = sub.add_parser("cab")
    p.add_argument("--algo", choices=CAB_ALGOS, default="homotopy")
    p.add_argument("--matrix", required=True)
    p.add_argument("--rhs", required=True)
    _config_flags(p)
    p.add_argument("--e-weight", dest="e_weight", type=float, default=None)
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_cab)

    p = sub.add_parser("align")
    p.add_argument("--algo", choices=("gp", "homotopy", "ist", "palm"), default="palm")
    p.add_argument("--basis", required=True)
    p.add_argument("--rhs", required=True)
    _config_flags(p)
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_align)

    p = sub.add_parser("report")
    p.add_argument("rest", nargs=argparse.REMAINDER)
    p.set_defaults(func=cmd_unsupported)
    return top


def run(argv):
    """One subcommand; returns the exit code (cli.py:574-592 conventions)."""
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:
        return 0 if exc.code in (0, None) else 2
    try:
        return args.func(args)
    except UsageError as exc:
        print("error: %s" % exc, file=sys.stderr)
        return 2
    except NumericalError as exc:
        print("solver failure: %s" % exc, file=sys.stderr)
        return 1
    except DeviceError as exc:
        print("device failure: %s" % exc, file=sys.stderr)
        return 2
    except ValueError as exc:
        print("error: %s" % exc, file=sys.stderr)
        return 2


def main():
    sys.exit(run(sys.argv[1:]))


if __name__ == "__main__":
    main()
