"""Golden parity cases: inputs are rebuilt from seeds, outputs come from the
real reference (``make_golden.py``) and are committed as ``<id>.npz``.

Input recipes
  genspec  : reference ``synth.make_instance(GenSpec(n, d, k, seed, sigma))``
             (unit-norm x0), rebuilt with ``oracle.gaussian_dict`` etc.
  workload : SURVEY §8(d) recipe (N(0,1) x0), ``paper_1007_3753_b200.synth``.
  qr       : orthonormal Q from ``default_rng(seed)`` and b ~ N(0,1).
  cab      : Gaussian A (d x n, seed) and a sparse-plus-corruption b.
"""

import numpy as np

# name -> recipe
CASES = []


def _add(cid, recipe, solver, cfg=None, extra=None, size="small"):
    CASES.append(dict(id=cid, recipe=recipe, solver=solver, cfg=cfg or {},
                      extra=extra or {}, size=size))


def _gs(n, d, k, seed, sigma=0.0):
    return dict(kind="genspec", n=n, d=d, k=k, seed=seed, sigma=sigma)


def _wl(d, n, k, seed=0, noise_rel=0.0):
    return dict(kind="workload", d=d, n=n, k=k, seed=seed, noise_rel=noise_rel)


REL = ("relative-estimate", 1e-6)

# ---- small first-order cases (fast; every option path) --------------------
for s in (1400, 1401, 1402):
    _add("fista_small_%d" % s, _gs(40, 20, 1 + s % 5, s, 0.02), "fista",
         dict(lam_rel=0.05, tol=1e-7, max_iter=2000))
_add("fista_small_exactL", _gs(40, 20, 3, 1500, 0.02), "fista",
     dict(lam_rel=0.05, tol=1e-9, max_iter=3000,
          options={"exact_L": True, "continuation": False}))
_add("fista_small_relobj", _gs(40, 20, 3, 1501, 0.02), "fista",
     dict(lam_rel=0.05, tol=1e-9, max_iter=3000,
          stopping=("relative-objective", 1e-8)))
_add("fista_small_kktrule", _gs(40, 20, 3, 1502, 0.02), "fista",
     dict(lam_rel=0.05, tol=1e-12, max_iter=3000, stopping=("kkt-residual", 1e-6)))
_add("fista_small_gtrule", _gs(40, 20, 2, 1503, 0.0), "fista",
     dict(lam_rel=0.001, tol=1e-12, max_iter=3000,
          stopping=("ground-truth-distance", 1e-2)))
_add("fista_small_budget", _gs(40, 20, 3, 19, 0.05), "fista",
     dict(lam=0.05, max_iter=2))
_add("fista_small_noncont", _gs(60, 30, 4, 1504, 0.01), "fista",
     dict(lam_rel=0.02, tol=1e-8, max_iter=5000,
          options={"continuation": False, "L0": 0.5, "eta": 2.0}))
_add("fista_qr", dict(kind="qr", d=8, seed=31), "fista", dict(lam=0.25, tol=1e-9))

for s in (1200, 1201):
    _add("ist_small_%d" % s, _gs(40, 20, 1 + s % 5, s, 0.02), "ist",
         dict(lam_rel=0.05, tol=1e-8, max_iter=3000))
_add("ist_small_sched", _gs(40, 20, 3, 1202, 0.02), "ist",
     dict(lam_rel=0.05, tol=1e-8, max_iter=3000), extra=dict(schedule="flat"))
_add("ist_small_relobj", _gs(40, 20, 3, 21, 0.0), "ist",
     dict(lam_rel=0.1, tol=1e-6, stopping=("relative-objective", 0.5)),
     extra=dict(schedule="flat"))

for s in (1700, 1701):
    _add("palm_small_%d" % s, _gs(60, 30, 3, s, 0.0), "palm",
         dict(tol=1e-6, max_iter=3000))
    _add("dalm_small_%d" % s, _gs(60, 30, 3, s, 0.0), "dalm",
         dict(tol=1e-6, max_iter=3000))
_add("dalm_small_beta", _gs(60, 30, 3, 1702, 0.0), "dalm",
     dict(tol=1e-6, max_iter=3000, options={"beta": 0.3}))
_add("dalm_small_cg", _gs(60, 30, 3, 1703, 0.0), "dalm",
     dict(tol=1e-6, max_iter=3000, options={"y_cg_step": True}))
_add("palm_small_rel", _gs(60, 30, 3, 1704, 0.0), "palm",
     dict(tol=1e-9, max_iter=3000, stopping=REL))

for s in (1300, 1301):
    _add("gpsr_small_%d" % s, _gs(40, 20, 3, s, 0.02), "gpsr",
         dict(lam_rel=0.05, tol=1e-7, max_iter=3000))
    _add("tnipm_small_%d" % s, _gs(40, 20, 3, s, 0.02), "tnipm",
         dict(lam_rel=0.05, tol=1e-7, max_iter=200))
    _add("homotopy_small_%d" % s, _gs(40, 20, 3, s, 0.02), "homotopy",
         dict(lam_rel=0.01))

# ---- PDIPA: equality-constrained interior point -------
for s in (1600, 1601, 1602):
    _add("pdipa_small_%d" % s, _gs(40, 20, 1 + s % 4, s, 0.0), "pdipa", dict(tol=1e-6))
_add("pdipa_small_noisy", _gs(60, 30, 4, 1603, 0.02), "pdipa", dict(tol=1e-8))
_add("pdipa_small_budget", _gs(40, 20, 3, 1604, 0.0), "pdipa", dict(max_iter=2))
_add("pdipa_qr", dict(kind="qr", d=8, seed=33), "pdipa", dict(tol=1e-9))

# ---- BASELINE config 1: 500 x 1000, k=50, noiseless, lambda 1e-3, rel-est --
_add("cfg1_fista", _wl(500, 1000, 50), "fista",
     dict(lam=1e-3, tol=1e-6, stopping=REL), size="cfg1")
_add("cfg1_palm", _wl(500, 1000, 50), "palm",
     dict(tol=1e-6, stopping=REL), size="cfg1")
_add("cfg1_dalm", _wl(500, 1000, 50), "dalm",
     dict(tol=1e-6, stopping=REL), size="cfg1")
_add("cfg1_dalm_native", _wl(500, 1000, 50), "dalm",
     dict(tol=1e-6), size="cfg1")
_add("cfg1_pdipa", _wl(500, 1000, 50), "pdipa", dict(tol=1e-6), size="cfg1")

# ---- BASELINE config 2: 1024 x 4096, k=128, 1% noise, default lambda -------
_cfg2 = _wl(1024, 4096, 128, 0, 0.01)
_add("cfg2_fista", _cfg2, "fista", dict(tol=1e-6, stopping=REL), size="cfg2")
_add("cfg2_fista_native", _cfg2, "fista", dict(tol=1e-6), size="cfg2")
_add("cfg2_ist", _cfg2, "ist", dict(tol=1e-6, stopping=REL), size="cfg2")
_add("cfg2_gpsr", _cfg2, "gpsr", dict(tol=1e-6, stopping=REL), size="cfg2")
_add("cfg2_tnipm", _cfg2, "tnipm", dict(tol=1e-6, stopping=REL), size="cfg2")
_add("cfg2_homotopy", _cfg2, "homotopy", dict(), size="cfg2")
_add("cfg2_palm", _cfg2, "palm", dict(tol=1e-6, stopping=REL), size="cfg2")
_add("cfg2_dalm_budget", _cfg2, "dalm", dict(tol=1e-6, max_iter=200), size="cfg2")
_add("cfg2_pdipa", _cfg2, "pdipa", dict(tol=1e-6), size="cfg2")

# ---- config-5 shape: 512 x 2048, lambda 1e-3 -------------------------------
for k in (16, 64):
    _add("cfg5_fista_k%d" % k, _wl(512, 2048, k, 5), "fista",
         dict(lam=1e-3, tol=1e-6, stopping=REL), size="cfg5")
    _add("cfg5_dalm_k%d" % k, _wl(512, 2048, k, 5), "dalm",
         dict(tol=1e-6, stopping=REL), size="cfg5")
    _add("cfg5_homotopy_k%d" % k, _wl(512, 2048, k, 5), "homotopy",
         dict(lam=1e-3), size="cfg5")

# ---- CAB ([A, I]) small ----------------------------------------------------
for solver in ("dalm", "fista", "pdipa"):
    _add("cab_small_%s" % solver, dict(kind="cab", d=40, n=30, k=3, seed=7, m=4),
         "cab:" + solver, dict(tol=1e-6, max_iter=5000))


def build_inputs(recipe):
    """Rebuild (A, b, ground_truth) from a recipe.  Uses only numpy and the
    oracle / product generators, so it runs on the GPU box as well."""
    kind = recipe["kind"]
    if kind == "genspec":
        from oracle import gaussian_dict, sparse_signal, with_noise
        A = gaussian_dict(recipe["d"], recipe["n"], recipe["seed"])
        x0 = sparse_signal(recipe["n"], recipe["k"], recipe["seed"])
        b = A @ x0
        if recipe["sigma"] > 0:
            b = with_noise(b, recipe["sigma"], recipe["seed"])
        return A, b, x0
    if kind == "workload":
        from paper_1007_3753_b200 import synth
        w = synth.Workload("golden", recipe["d"], recipe["n"], recipe["k"],
                           recipe["seed"], recipe["noise_rel"])
        P = synth.make_problem(w)
        return P.A, P.b, P.ground_truth
    if kind == "qr":
        rng = np.random.default_rng(recipe["seed"])
        Q, _ = np.linalg.qr(rng.standard_normal((recipe["d"], recipe["d"])))
        b = rng.standard_normal(recipe["d"])
        return Q, b, None
    if kind == "cab":
        from oracle import corrupt, gaussian_dict
        A = gaussian_dict(recipe["d"], recipe["n"], recipe["seed"])
        rng = np.random.default_rng(recipe["seed"] + 9)
        x0 = np.zeros(recipe["n"])
        x0[rng.choice(recipe["n"], recipe["k"], replace=False)] = rng.standard_normal(recipe["k"])
        b, _ = corrupt(A @ x0, recipe["m"] / recipe["d"], -1.0, 1.0, recipe["seed"])
        return A, b, x0
    raise ValueError(kind)


def resolve_lambda(cfg, A, b):
    if "lam" in cfg:
        return cfg["lam"]
    if "lam_rel" in cfg:
        return cfg["lam_rel"] * float(np.max(np.abs(A.T @ b)))
    return None


def get(cid):
    for c in CASES:
        if c["id"] == cid:
            return c
    raise KeyError(cid)
