"""Seeded alignment instances (tall B with a few grossly corrupted rows) and
the solver settings of the alignment golden cases."""

import numpy as np


def align_instance(seed, d, m, frac=0.1, amp=3.0):
    """b = B w0 + e0: B iid N(0,1) (d x m), w0 N(0,1), e0 nonzero on
    round(frac d) random rows with uniform(-amp, amp) values."""
    rng = np.random.default_rng(np.random.SeedSequence((seed, 17)))
    B = rng.standard_normal((d, m))
    w0 = rng.standard_normal(m)
    e0 = np.zeros(d)
    rows = rng.choice(d, int(round(frac * d)), replace=False)
    e0[rows] = rng.uniform(-amp, amp, rows.size)
    return B, B @ w0 + e0


CASES = {
    "palm_120x11": {"solver": "palm", "recipe": dict(seed=1, d=120, m=11), "tol": 1e-10, "max_iter": 5000},
    "palm_60x7": {"solver": "palm", "recipe": dict(seed=2, d=60, m=7), "tol": 1e-8, "max_iter": 5000},
    "palm_1024x11": {"solver": "palm", "recipe": dict(seed=3, d=1024, m=11, frac=0.2), "tol": 1e-8,
                     "max_iter": 5000},
    "palm_mu": {"solver": "palm", "recipe": dict(seed=4, d=200, m=16), "tol": 1e-9, "max_iter": 5000,
                "options": {"mu0": 0.5, "rho": 1.5}},
    "palm_budget": {"solver": "palm", "recipe": dict(seed=5, d=80, m=5), "tol": 1e-12, "max_iter": 37},
    "ist_60x7": {"solver": "ist", "recipe": dict(seed=6, d=60, m=7), "tol": 1e-9, "max_iter": 20000},
    "hom_120x11": {"solver": "homotopy", "recipe": dict(seed=8, d=120, m=11), "tol": 1e-9, "max_iter": 5000},
    "hom_60x7_lam": {"solver": "homotopy", "recipe": dict(seed=9, d=60, m=7), "tol": 1e-8, "max_iter": 5000,
                     "lam": 0.02},
    "hom_1024x11": {"solver": "homotopy", "recipe": dict(seed=10, d=1024, m=11, frac=0.2), "tol": 1e-8,
                    "max_iter": 5000},
    "gp_120x11": {"solver": "gp", "recipe": dict(seed=11, d=120, m=11), "tol": 1e-8, "max_iter": 200},
    "gp_60x7_lam": {"solver": "gp", "recipe": dict(seed=12, d=60, m=7), "tol": 1e-9, "max_iter": 200, "lam": 0.1},
    "gp_512x8": {"solver": "gp", "recipe": dict(seed=13, d=512, m=8, frac=0.15), "tol": 1e-8, "max_iter": 200},
    "ist_120x11_lam": {"solver": "ist", "recipe": dict(seed=7, d=120, m=11), "tol": 1e-8, "max_iter": 20000,
                       "lam": 0.05},
}
