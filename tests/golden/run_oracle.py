"""Run a golden case through the oracle (test infrastructure)."""

import numpy as np

import oracle
from tests.golden.cases import build_inputs, resolve_lambda


def run_oracle(case):
    A, b, gt = build_inputs(case["recipe"])
    cfg = case["cfg"]
    lam = resolve_lambda(cfg, A, b)
    kw = dict(tol=cfg.get("tol", 1e-6), max_iter=cfg.get("max_iter", 5000),
              stop=cfg.get("stopping"))
    opts = dict(cfg.get("options", {}))
    s = case["solver"]
    extra = {}
    if s.startswith("cab:"):
        x, e, res = oracle.cab(A, b, s[4:], lam=lam, opts=opts, **kw)
        extra["e"] = e
        return res, x, extra
    if s == "fista":
        res = oracle.fista(A, b, lam=lam, opts=opts, gt=gt, **kw)
    elif s == "ist":
        stages = None
        if case["extra"].get("schedule") == "flat":
            stages = oracle.schedule_stages(lam, 0.5, lam)
        res = oracle.ist(A, b, stages=stages, lam=lam, gt=gt, **kw)
    elif s == "palm":
        res = oracle.palm(A, b, opts=opts, gt=gt, **kw)
    elif s == "dalm":
        res = oracle.dalm(A, b, opts=opts, gt=gt, **kw)
    elif s == "gpsr":
        res = oracle.gpsr(A, b, lam=lam, gt=gt, **kw)
    elif s == "tnipm":
        res = oracle.tnipm(A, b, lam=lam, opts=opts, gt=gt, **kw)
    elif s == "homotopy":
        target = lam if lam is not None else 1e-2 * float(np.max(np.abs(A.T @ b)))
        res, _ = oracle.homotopy(A, b, target, max_iter=kw["max_iter"])
    elif s == "pdipa":
        res = oracle.pdipa(A, b, gt=gt, **kw)
    else:
        raise ValueError(s)
    return res, res.x, extra


def load_golden(cid):
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    z = np.load(os.path.join(here, cid + ".npz"))
    return {k: z[k] for k in z.files}
