"""Pin the CPU oracle against the real reference's golden outputs.

The fixtures under tests/golden/ were produced by running the unmodified
reference package (compiled _accel) on seed-rebuilt inputs
(tests/golden/make_golden.py).  The oracle restatement must reproduce them:
identical iteration counts / convergence flags / notes and traces, iterates
to 1e-12 relative (bitwise on the same BLAS in practice).
"""

import json

import numpy as np
import pytest

import oracle
from tests.golden.cases import CASES
from tests.golden.run_oracle import load_golden, run_oracle

FAST = [c["id"] for c in CASES if c["size"] in ("small", "cfg1", "cfg5")
        and c["id"] not in ("cfg1_dalm_native",)]
SLOW = [c["id"] for c in CASES if c["id"] not in FAST]


def _check(cid):
    case = next(c for c in CASES if c["id"] == cid)
    gold = load_golden(cid)
    res, x, extra = run_oracle(case)
    assert res.iterations == int(gold["iterations"])
    assert bool(res.converged) == bool(gold["converged"])
    assert list(res.notes) == json.loads(str(gold["notes"]))
    ref = gold["x"]
    scale = max(np.linalg.norm(ref), 1e-300)
    assert np.linalg.norm(x - ref) <= 1e-12 * scale
    tr = np.array(res.trace, dtype=np.float64).reshape(-1, 4)
    assert tr.shape == gold["trace"].shape
    np.testing.assert_array_equal(tr[:, 0], gold["trace"][:, 0])
    np.testing.assert_array_equal(tr[:, 3], gold["trace"][:, 3])
    np.testing.assert_allclose(tr[:, 1:3], gold["trace"][:, 1:3], rtol=1e-11, atol=1e-300)
    if "e" in gold:
        np.testing.assert_allclose(extra["e"], gold["e"], rtol=0, atol=1e-12 * scale)


@pytest.mark.parametrize("cid", FAST)
def test_oracle_matches_reference(cid):
    _check(cid)


@pytest.mark.slow
@pytest.mark.parametrize("cid", SLOW)
def test_oracle_matches_reference_large(cid):
    _check(cid)


# ---- unit known-answer tests from the reference's own suite ---------------

def test_t_next_frozen_values():
    # test_shrinkage.py:79-82
    assert oracle.t_next(1.0) == pytest.approx(1.6180339887498949, rel=1e-15)
    assert oracle.t_next(1.6180339887498949) == pytest.approx(2.193527085331054, rel=1e-12)


def test_t_next_momentum_inequality():
    t = 1.0
    for _ in range(3000):
        tn = oracle.t_next(t)
        assert tn * tn - tn <= t * t
        t = tn


def test_backtrack_scalar_case():
    # test_shrinkage.py:125-128
    L, _ = oracle.backtrack(np.array([[2.0]]), np.array([2.0]), np.array([0.0]), 1.0, 2.0, 0.0)
    assert L == 4.0


def test_bb_alpha_examples():
    # test_shrinkage.py:19-28
    assert oracle.bb(np.array([1.0, 1.0]), np.array([2.0, 4.0])) == 3.0
    assert oracle.bb(np.array([1.0, 0.0]), np.array([0.0, 1.0])) == 1e-30
    assert oracle.bb(np.array([1e-20, 0.0]), np.array([1e20, 0.0])) == 1e30


def test_soft_threshold_examples():
    # test_numerics.py:20-35
    out = oracle.soft(np.array([3.0, -3.0, 0.5, -0.5, 1.0]), 1.0)
    np.testing.assert_array_equal(out, [2.0, -2.0, 0.0, 0.0, 0.0])


def test_homotopy_gamma_frozen_cases():
    # test_homotopy.py:112-123 frozen gammas on a seeded instance
    rng = np.random.default_rng(5)
    n = 16
    c = rng.uniform(-1, 1, n)
    x = np.zeros(n)
    mask = np.zeros(n, dtype=bool)
    mask[[1, 12]] = True
    x[mask] = rng.standard_normal(2)
    d = np.zeros(n)
    d[mask] = rng.standard_normal(2)
    w = rng.uniform(-0.5, 0.5, n)
    gp, ip, gm, im = oracle.step_lengths(1.0, c, x, d, w, mask)
    # exhaustive enumeration
    best = (np.inf, -1)
    for j in range(n):
        if mask[j]:
            continue
        for r in ((1.0 - c[j]) / (1.0 - w[j]), (1.0 + c[j]) / (1.0 + w[j])):
            if np.isfinite(r) and r > 1e-10 and r < best[0]:
                best = (r, j)
    assert (gp, ip) == best


def test_rank1_update_downdate_roundtrip():
    rng = np.random.default_rng(3)
    B = rng.standard_normal((6, 6))
    R = oracle.chol_upper(B @ B.T + 6 * np.eye(6))
    v = rng.standard_normal(6)
    R2 = R.copy()
    oracle.rank1_update(R2, v.copy())
    np.testing.assert_allclose(R2.T @ R2, R.T @ R + np.outer(v, v), atol=1e-10)
    assert oracle.rank1_downdate(R2, v.copy()) == 0
    np.testing.assert_allclose(R2.T @ R2, R.T @ R, atol=1e-9)
