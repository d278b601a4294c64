"""Experiment harness on the B200: phase grids, noise sweeps, corruption
sweeps — the reference's ell1.bench API (bench.py:64-335) with every trial of
an experiment solved in group launches (paper_1007_3753_b200.group).

Same contract as the reference: each trial's instance comes from
(base_seed, grid indices, trial index) through synth.trial_seed, so the same
configuration reproduces the same instances and every solver of a comparison
sees identical data; success / error / iteration columns are deterministic
(fixed-order device reductions), wall times are not.  ``jobs`` is accepted
for signature compatibility and ignored: one device runs all trials of an
experiment concurrently.  Reported wall time per trial = the group's solve
time divided by its trial count (generation and I/O excluded, as in the
reference).  PDIPA has no group form; its trials run one solve at a time.
"""

import csv
import json
import platform
from dataclasses import dataclass

import numpy as np

from paper_1007_3753_b200.group import GROUP_SOLVERS, TrialGroup
from paper_1007_3753_b200.model import ProblemInstance, SolverConfig
from paper_1007_3753_b200.synth import (RNG_NAME, GenSpec, add_noise, corrupt_entries, gen_bouquet_dict,
                                        gen_gaussian_dict, gen_sparse_signal, make_instance,
                                        trial_seed)

SOLVER_NAMES = ("pdipa", "homotopy", "gpsr", "tnipm", "ist", "fista", "palm", "dalm")
_PHASE_LAM_REL = 1e-4          # bench.py:36 — vanishing penalty for noiseless recovery


@dataclass(frozen=True)
class PhaseGrid:
    """Success rates over a sparsity-rate / sampling-rate grid (bench.py:65-95)."""

    n: int
    rho_values: tuple
    delta_values: tuple
    success_rate: np.ndarray
    trials_per_cell: int
    base_seed: int
    success_tol: float

    def __post_init__(self):
        for seq in (self.rho_values, self.delta_values):
            arr = np.asarray(seq, dtype=np.float64)
            if arr.size == 0 or np.any(arr <= 0.0) or np.any(arr > 1.0):
                raise ValueError("grid axes must lie in (0, 1]")
            if np.any(np.diff(arr) <= 0.0):
                raise ValueError("grid axes must be strictly increasing")
        rates = np.asarray(self.success_rate, dtype=np.float64)
        if rates.shape != (len(self.rho_values), len(self.delta_values)):
            raise ValueError("success_rate shape must be |rho| x |delta|")
        if np.any(rates < 0.0) or np.any(rates > 1.0):
            raise ValueError("success rates must lie in [0, 1]")
        if self.trials_per_cell < 1:
            raise ValueError("trials_per_cell must be at least 1")
        if not self.success_tol > 0:
            raise ValueError("success_tol must be positive")


@dataclass(frozen=True)
class SweepResult:
    """Per-solver metrics along one axis, |solvers| x |axis| (bench.py:98-124)."""

    axis_name: str
    axis_values: tuple
    solvers: tuple
    trials: int
    mean_time: np.ndarray
    mean_rel_error: np.ndarray = None
    mean_iterations: np.ndarray = None
    success_rate: np.ndarray = None

    def __post_init__(self):
        if self.trials < 1:
            raise ValueError("trials must be at least 1")
        want = (len(self.solvers), len(self.axis_values))
        for name in ("mean_time", "mean_rel_error", "mean_iterations", "success_rate"):
            mat = getattr(self, name)
            if mat is not None and np.asarray(mat).shape != want:
                raise ValueError("%s must be |solvers| x |axis|" % name)


def _solve_all(name, problems, cfg, lams, ext=False, group=None):
    """Solve every trial with one solver; returns SolverResults in order."""
    if name == "gp":
        name = "gpsr"
    if name not in SOLVER_NAMES:
        raise ValueError("unknown solver %r (choose from %s)" % (name, ", ".join(SOLVER_NAMES)))
    if name in GROUP_SOLVERS:
        grp = group if group is not None else TrialGroup(problems, ext=ext)
        return grp.solve(name, cfg, lams=lams)
    from paper_1007_3753_b200.solvers import solve_named
    out = []
    for i, P in enumerate(problems):
        c = SolverConfig(lam=None if lams is None else float(lams[i]), tol=cfg.tol,
                         max_iter=cfg.max_iter, stopping=cfg.stopping, options=dict(cfg.options))
        out.append(solve_named(name, P, c))
    return out


def run_phase_grid(solver, n, rho_values, delta_values, trials, success_tol=1e-3, base_seed=0,
                   config=None, jobs=1):
    """Success-rate grid over rho = k/n, delta = d/n (bench.py:154-190):
    k = round(rho n), d = round(delta n) per cell, `trials` instances each,
    success = relative l2 error <= success_tol; penalised solvers run at
    1e-4 ||A^T b||_inf unless config.lam pins a weight."""
    if trials < 1:
        raise ValueError("trials must be at least 1")
    tol = config.tol if config is not None else 1e-8
    max_iter = config.max_iter if config is not None else 20000
    lam = config.lam if config is not None else None
    problems = []
    for i, rho in enumerate(rho_values):
        for j, delta in enumerate(delta_values):
            k = max(1, int(round(rho * n)))
            d = max(1, int(round(delta * n)))
            for t in range(trials):
                problems.append(make_instance(GenSpec(n=n, d=d, k=k, seed=trial_seed(base_seed, i, j, t))))
    grp = TrialGroup(problems)
    lams = np.full(len(problems), float(lam)) if lam is not None else _PHASE_LAM_REL * grp.correlation_max()
    cfg = SolverConfig(tol=tol, max_iter=max_iter)
    res = _solve_all(solver, problems, cfg, lams, group=grp)
    flags = [float(np.linalg.norm(r.x_star - P.ground_truth)) <= success_tol * float(np.linalg.norm(P.ground_truth))
             for r, P in zip(res, problems)]
    rates = np.asarray(flags, dtype=np.float64).reshape(len(rho_values), len(delta_values), trials).mean(axis=2)
    return PhaseGrid(n=n, rho_values=tuple(float(r) for r in rho_values),
                     delta_values=tuple(float(x) for x in delta_values), success_rate=rates,
                     trials_per_cell=trials, base_seed=base_seed, success_tol=success_tol)


def interpolate_success_contour(grid, level):
    """First downward crossing of `level` per delta column, linearly
    interpolated in rho (bench.py:193-215); [(delta, rho), ...]."""
    if not 0.0 < level < 1.0:
        raise ValueError("level must lie in (0, 1)")
    rho = np.asarray(grid.rho_values)
    out = []
    for j, delta in enumerate(grid.delta_values):
        col = grid.success_rate[:, j]
        for i in range(len(rho) - 1):
            hi, lo = col[i], col[i + 1]
            if hi >= level > lo:
                frac = (hi - level) / (hi - lo)
                out.append((float(delta), float(rho[i] + frac * (rho[i + 1] - rho[i]))))
                break
    return out


def run_noise_sweep(solvers, mode, spec, trials, base_seed=0, config=None, jobs=1):
    """Noisy recovery along d ("vary-d": spec n, k, d_values) or rho
    ("vary-k": spec n, d, rho_values), all solvers on the same instances
    (bench.py:243-285): signals sqrt(k)-scaled, noise_sigma default 0.1,
    lambda = noise_sigma (or 1e-4 ||A^T b||_inf noise-free) unless config.lam."""
    if trials < 1:
        raise ValueError("trials must be at least 1")
    if mode not in ("vary-d", "vary-k"):
        raise ValueError("mode must be vary-d or vary-k")
    solvers = tuple(solvers)
    n = int(spec["n"])
    sigma = float(spec.get("noise_sigma", 0.1))
    if mode == "vary-d":
        axis = tuple(int(v) for v in spec["d_values"])
        cells = [(int(spec["k"]), d) for d in axis]
    else:
        axis = tuple(float(v) for v in spec["rho_values"])
        cells = [(max(1, int(round(r * n))), int(spec["d"])) for r in axis]
    tol = config.tol if config is not None else 1e-6
    max_iter = config.max_iter if config is not None else 5000
    lam = config.lam if config is not None else None
    problems = []
    for i, (k, d) in enumerate(cells):
        for t in range(trials):
            seed = trial_seed(base_seed, i, t)
            A = gen_gaussian_dict(d, n, seed)
            x0 = np.sqrt(k) * gen_sparse_signal(n, k, seed)
            b = add_noise(A @ x0, sigma, seed)
            problems.append(ProblemInstance(A, b, ground_truth=x0, noise_sigma=sigma))
    grp = TrialGroup(problems)
    if lam is not None:
        lams = np.full(len(problems), float(lam))
    elif sigma == 0.0:
        lams = _PHASE_LAM_REL * grp.correlation_max()
    else:
        lams = np.full(len(problems), sigma)
    cfg = SolverConfig(tol=tol, max_iter=max_iter)
    data = np.zeros((len(problems), len(solvers), 3))
    for s, name in enumerate(solvers):
        res = _solve_all(name, problems, cfg, lams, group=grp)
        for q, (r, P) in enumerate(zip(res, problems)):
            err = float(np.linalg.norm(r.x_star - P.ground_truth) / np.linalg.norm(P.ground_truth))
            data[q, s] = (r.wall_time_seconds, err, r.iterations)
    means = data.reshape(len(axis), trials, len(solvers), 3).mean(axis=1)
    return SweepResult(axis_name="d" if mode == "vary-d" else "rho", axis_values=axis, solvers=solvers,
                       trials=trials, mean_time=means[:, :, 0].T, mean_rel_error=means[:, :, 1].T,
                       mean_iterations=means[:, :, 2].T)


def run_corruption_sweep(dict_spec, corruption_levels, solvers, trials, base_seed=0, config=None, jobs=1):
    """Group identification under gross corruption (bench.py:288-335): one
    planted group of a bouquet dictionary, `level` of the measurements
    replaced, each backend solves the [A, I] extension (robust.cab_solve);
    a hit = the planted group carries the most coefficient energy."""
    if trials < 1:
        raise ValueError("trials must be at least 1")
    solvers = tuple(solvers)
    d, n = int(dict_spec["d"]), int(dict_spec["n"])
    groups = int(dict_spec["groups"])
    coherence = float(dict_spec["coherence"])
    amp = float(dict_spec.get("corruption_amp", 1.0))
    levels = tuple(float(v) for v in corruption_levels)
    tol = config.tol if config is not None else 1e-8
    max_iter = config.max_iter if config is not None else 4000
    problems, planted, labels_of = [], [], []
    for i, lv in enumerate(levels):
        for t in range(trials):
            seed = trial_seed(base_seed, i, t)
            rng = np.random.default_rng(seed)
            A, labels = gen_bouquet_dict(d, n, groups, coherence, seed)
            g = int(rng.integers(groups))
            members = np.flatnonzero(labels == g)
            active = rng.choice(members, size=min(3, members.size), replace=False)
            x0 = np.zeros(n)
            x0[active] = rng.uniform(0.5, 1.5, size=active.size) * rng.choice([-1.0, 1.0], size=active.size)
            b = A @ x0
            scale = amp * float(np.max(np.abs(b)))
            b_bad, _ = corrupt_entries(b, lv, -scale, scale, seed + 100000)
            problems.append(ProblemInstance(A, b_bad))
            planted.append(g)
            labels_of.append(labels)
    from paper_1007_3753_b200.robust import _CAB_BACKENDS
    for name in solvers:
        if name not in _CAB_BACKENDS:
            raise ValueError("unknown cab backend %r (choose from %s)" % (name, ", ".join(_CAB_BACKENDS)))
    cfg = SolverConfig(tol=tol, max_iter=max_iter)
    grp = TrialGroup(problems, ext=True)
    data = np.zeros((len(problems), len(solvers), 2))
    for s, name in enumerate(solvers):
        lams = None
        key = "gpsr" if name == "gp" else name
        if key in ("gpsr", "homotopy"):
            lams = 1e-2 * grp.correlation_max()            # robust.py:_resolved_lambda on [A, I]
        if key in GROUP_SOLVERS:
            res = grp.solve(key, cfg, lams=lams)
            xs = [r.x_star[:n] for r in res]
            times = [r.wall_time_seconds for r in res]
        else:
            import time
            from paper_1007_3753_b200.robust import cab_solve
            xs, times = [], []
            for P in problems:
                t0 = time.perf_counter()
                x, _, _ = cab_solve(P.A, P.b, name, cfg)
                times.append(time.perf_counter() - t0)
                xs.append(x)
        for q, x in enumerate(xs):
            lab = labels_of[q]
            norms = [np.linalg.norm(x[lab == gg]) for gg in range(groups)]
            data[q, s] = (times[q], float(int(np.argmax(norms)) == planted[q]))
    means = data.reshape(len(levels), trials, len(solvers), 2).mean(axis=1)
    return SweepResult(axis_name="corruption", axis_values=levels, solvers=solvers, trials=trials,
                       mean_time=means[:, :, 0].T, success_rate=means[:, :, 1].T)


def _fmt(v):
    return "%.17g" % float(v)


def phase_grid_to_csv(grid, path):
    """rho, delta, success_rate per cell (bench.py:342-352); deterministic."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["rho", "delta", "success_rate"])
        for i, rho in enumerate(grid.rho_values):
            for j, delta in enumerate(grid.delta_values):
                w.writerow([_fmt(rho), _fmt(delta), _fmt(grid.success_rate[i, j])])
    return path


def sweep_to_csv(sweep, path):
    """One row per (axis value, solver) with the metrics present (bench.py:355-381)."""
    metrics = [(name, getattr(sweep, name)) for name in
               ("mean_time", "mean_rel_error", "mean_iterations", "success_rate")
               if getattr(sweep, name) is not None]
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        header = [sweep.axis_name, "solver"]
        for name, _ in metrics:
            header.append("mean_time_seconds" if name == "mean_time" else name)
        w.writerow(header)
        for j, val in enumerate(sweep.axis_values):
            for s, solver in enumerate(sweep.solvers):
                row = [_fmt(val), solver]
                row.extend(_fmt(mat[s, j]) for _, mat in metrics)
                w.writerow(row)
    return path


def environment_metadata():
    """Reproducibility context (bench.py:384-393)."""
    import paper_1007_3753_b200
    from paper_1007_3753_b200 import _lib
    return {"package_version": getattr(paper_1007_3753_b200, "__version__", "0"),
            "python": platform.python_version(), "numpy": np.__version__, "rng": RNG_NAME,
            "platform": platform.platform(), "compiled_kernels": _lib.lib().ell1_version().decode()}


def write_summary_json(path, kind, parameters, results=None):
    """Stable-key JSON summary (bench.py:396-407)."""
    payload = {"kind": kind, "parameters": parameters, "environment": environment_metadata()}
    if results is not None:
        payload["results"] = results
    with open(path, "w") as fh:
        json.dump(payload, fh, sort_keys=True, indent=2)
        fh.write("\n")
    return path
