"""Shared helpers for the -m gpu parity tests."""

import json

import numpy as np

from tests.golden.cases import CASES, build_inputs, resolve_lambda
from tests.golden.run_oracle import load_golden


def rel_err(x, ref):
    den = float(np.linalg.norm(ref))
    if den == 0.0:
        return float(np.linalg.norm(x))
    return float(np.linalg.norm(x - ref)) / den


def support(x, rel=1e-3):
    m = float(np.max(np.abs(x))) if x.size else 0.0
    return set(np.nonzero(np.abs(x) > rel * m)[0].tolist()) if m > 0 else set()


def assert_parity(res_x, iterations, converged, trace, gold, rtol, iter_slack=0,
                  check_trace=True, trace_atol=1e-12):
    """North-star gates: rel l2 error, identical support at 1e-3 max|x|,
    same convergence flag and iteration count (optionally within slack)."""
    ref = gold["x"]
    err = rel_err(res_x, ref)
    assert err <= rtol, "relative error %.3e > %.1e" % (err, rtol)
    assert support(res_x) == support(ref), "support differs"
    assert bool(converged) == bool(gold["converged"])
    assert abs(int(iterations) - int(gold["iterations"])) <= iter_slack, \
        "iterations %d vs reference %d" % (iterations, int(gold["iterations"]))
    if check_trace and iter_slack == 0:
        tr = np.array([tuple(t) for t in trace], dtype=np.float64).reshape(-1, 4)
        g = gold["trace"]
        assert tr.shape == g.shape
        np.testing.assert_array_equal(tr[:, 0], g[:, 0])
        np.testing.assert_allclose(tr[:, 1:3], g[:, 1:3], rtol=max(rtol, 1e-9), atol=trace_atol)


def case_inputs(cid):
    case = next(c for c in CASES if c["id"] == cid)
    A, b, gt = build_inputs(case["recipe"])
    return case, A, b, gt, load_golden(cid)


def make_config(case, A, b, dtype="float64", **over):
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    cfg = case["cfg"]
    lam = resolve_lambda(cfg, A, b)
    stop = cfg.get("stopping")
    opts = dict(cfg.get("options", {}))
    opts["dtype"] = dtype
    kw = dict(lam=lam, tol=cfg.get("tol", 1e-6), max_iter=cfg.get("max_iter", 5000),
              stopping=StoppingRule(*stop) if stop else None, options=opts)
    kw.update(over)
    return SolverConfig(**kw)


def ids_for(solver, sizes=("small", "cfg1", "cfg2", "cfg5")):
    return [c["id"] for c in CASES if c["solver"] == solver and c["size"] in sizes]


def gold_notes(gold):
    return tuple(json.loads(str(gold["notes"])))
