"""Alignment solvers batched across images (robust.py:223-515)
against the reference's own outputs (tests/golden/make_align_golden.py), plus
the reference's edge cases (test_robust.py: rank-deficient basis, zero data,
option validation).  Batched element j must equal the single-image call."""

import os

import numpy as np
import pytest

from tests.golden.align_cases import CASES, align_instance

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "align_golden.npz")


def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _rel(x, ref):
    return float(np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.mark.parametrize("name", sorted(CASES))
def test_align_matches_reference(name):
    _cuda()
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.robust import (AlignmentProblem, align_gp_solve, align_homotopy_solve,
                                             align_ist_solve, align_palm_solve)
    c = CASES[name]
    gold = np.load(GOLD)
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
    assert _rel(w, gold[name + "_w"]) <= 1e-6
    assert _rel(e, gold[name + "_e"]) <= 1e-6
    top = np.max(np.abs(gold[name + "_e"]))
    assert set(np.nonzero(np.abs(e) > 1e-3 * top)[0]) == set(np.nonzero(np.abs(gold[name + "_e"]) > 1e-3 * top)[0])


@pytest.mark.parametrize("solver", ["palm", "ist", "homotopy", "gp"])
def test_batch_equals_single_images(solver):
    _cuda()
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200 import robust
    insts = [align_instance(seed=100 + j, d=150, m=9) for j in range(12)]
    Bs = np.stack([B for B, _ in insts])
    bs = np.stack([b for _, b in insts])
    cfg = SolverConfig(tol=1e-8, max_iter=5000)
    if solver == "palm":
        W, E = robust.align_palm_solve_batch(Bs, bs, cfg)
    elif solver == "homotopy":
        W, E = robust.align_homotopy_solve_batch(Bs, bs, cfg)
    elif solver == "gp":
        W, E = robust.align_gp_solve_batch(Bs, bs, None, cfg)
    else:
        W, E = robust.align_ist_solve_batch(Bs, bs, None, cfg)
    for j, (B, b) in enumerate(insts):
        prob = robust.AlignmentProblem(B, b)
        if solver == "palm":
            w, e = robust.align_palm_solve(prob, cfg)
        elif solver == "homotopy":
            w, e = robust.align_homotopy_solve(prob, cfg)
        elif solver == "gp":
            w, e = robust.align_gp_solve(prob, None, cfg)
        else:
            w, e = robust.align_ist_solve(prob, None, cfg)
        assert np.array_equal(W[j], w) and np.array_equal(E[j], e)


def test_rank_deficient_basis_raises():
    _cuda()
    from paper_1007_3753_b200.exceptions import IllConditionedError
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.robust import AlignmentProblem, align_ist_solve, align_palm_solve
    B, b = align_instance(seed=9, d=40, m=4)
    B[:, 3] = 0.0                      # zero column: G has a zero pivot (the reference raises too)
    prob = AlignmentProblem(B, b)
    with pytest.raises(IllConditionedError):
        align_palm_solve(prob, SolverConfig())
    with pytest.raises(IllConditionedError):
        align_ist_solve(prob, 0.1, SolverConfig())
    from paper_1007_3753_b200.robust import align_gp_solve
    with pytest.raises(IllConditionedError):
        align_gp_solve(prob, 0.1, SolverConfig())


def test_zero_data_and_option_validation():
    _cuda()
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.robust import AlignmentProblem, align_ist_solve, align_palm_solve
    B, _ = align_instance(seed=10, d=30, m=3)
    w, e = align_palm_solve(AlignmentProblem(B, np.zeros(30)), SolverConfig())
    assert np.all(w == 0.0) and np.all(e == 0.0)
    prob = AlignmentProblem(B, B @ np.ones(3))
    with pytest.raises(ValueError):
        align_palm_solve(prob, SolverConfig(options={"mu0": 0.0}))
    with pytest.raises(ValueError):
        align_palm_solve(prob, SolverConfig(options={"rho": 1.0}))
    with pytest.raises(ValueError):
        align_ist_solve(prob, -1.0, SolverConfig())


def test_ist_block_step_matches_reference_formula():
    """robust.ist_block_step (robust.py:433-445) on the device vs the
    reference's numpy expression; alpha <= 0 raises ValueError."""
    _cuda()
    from paper_1007_3753_b200.robust import ist_block_step
    from oracle.l1_oracle import soft
    rng = np.random.default_rng(5)
    for d, m in ((40, 3), (1500, 11), (5000, 32)):
        B = rng.standard_normal((d, m))
        b, e, w = rng.standard_normal(d), rng.standard_normal(d) * (rng.random(d) < 0.2), rng.standard_normal(m)
        lam, alpha = 0.3, 2.5
        wn, en = ist_block_step(B, b, w, e, lam, alpha)
        r = b - B @ w - e
        np.testing.assert_allclose(wn, w + (B.T @ r) / alpha, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(en, soft(e + r / alpha, lam / alpha), rtol=1e-12, atol=1e-12)
    with pytest.raises(ValueError):
        ist_block_step(B, b, w, e, lam, 0.0)


@pytest.mark.parametrize("d,m", [(1024, 32), (2048, 16), (2304, 8), (5000, 6)])
def test_align_large_images_stage_b_in_global_memory(d, m):
    """Images whose (d+1) m doubles exceed the SM's shared memory:
    B is staged in global memory; results equal the numpy PALM restatement."""
    _cuda()
    from oracle.l1_oracle import align_palm
    from paper_1007_3753_b200 import robust
    from paper_1007_3753_b200.model import SolverConfig
    insts = [align_instance(seed=900 + j, d=d, m=m, frac=0.2) for j in range(3)]
    Bs = np.stack([B for B, _ in insts])
    bs = np.stack([b for _, b in insts])
    cfg = SolverConfig(tol=1e-8, max_iter=5000)
    W, E = robust.align_palm_solve_batch(Bs, bs, cfg)
    for j in range(3):
        w_ref, e_ref = align_palm(Bs[j], bs[j], tol=1e-8, max_iter=5000)
        assert _rel(W[j], w_ref) <= 1e-9
        assert _rel(E[j], e_ref) <= 1e-9


@pytest.mark.parametrize("solver", ["palm", "ist", "homotopy", "gp"])
def test_large_image_variant_bit_identical(solver):
    """The large-image kernels (32 rows per thread, d <= 8192; ADVICE r01:
    the reference accepts any tall B) forced onto the golden cases give the
    same bits as the default variant: same row map and accumulation order."""
    _cuda()
    from paper_1007_3753_b200 import _lib, robust
    from paper_1007_3753_b200.model import SolverConfig
    insts = [align_instance(seed=700 + j, d=120, m=11, frac=0.1) for j in range(4)]
    Bs = np.stack([B for B, _ in insts])
    bs = np.stack([b for _, b in insts])
    cfg = SolverConfig(tol=1e-8, max_iter=5000)
    lam = 0.05 if solver in ("ist", "gp") else None
    L = _lib.lib()
    try:
        W0, E0, I0 = robust._align_batch(solver, Bs, bs, cfg, lam)
        L.ell1_test_align_large_rows(1)
        W1, E1, I1 = robust._align_batch(solver, Bs, bs, cfg, lam)
    finally:
        L.ell1_test_align_large_rows(0)
    assert np.array_equal(I0, I1)
    assert np.array_equal(W0, W1) and np.array_equal(E0, E1)
