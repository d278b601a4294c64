"""Host-side record logic of the boundary (no GPU): the reference's
test_model.py record/stop-rule scenarios restated against
paper_1007_3753_b200.model, plus the no-CPU-fallback guarantee."""

import numpy as np
import pytest

from paper_1007_3753_b200 import model
from paper_1007_3753_b200.model import (ProblemInstance, SolverConfig, SolverResult,
                                        StopRecord, StoppingRule)


def test_problem_instance_validation():
    with pytest.raises(ValueError):
        ProblemInstance(np.eye(3), np.zeros(2))
    with pytest.raises(ValueError):
        ProblemInstance(np.eye(3), np.zeros(3), ground_truth=np.zeros(2))
    with pytest.raises(ValueError):
        ProblemInstance(np.array([[np.inf, 0.0]]), np.zeros(1))
    P = ProblemInstance(np.eye(2), np.ones(2))
    assert P.d == 2 and P.n == 2


def test_solver_config_validation():
    for bad in ({"lam": -1.0}, {"tol": 0.0}, {"max_iter": 0}):
        with pytest.raises(ValueError):
            SolverConfig(**bad)
    assert SolverConfig().max_iter == 5000
    assert SolverConfig(lam=0.7).resolved_lambda(ProblemInstance(np.eye(2), np.ones(2))) == 0.7


def test_stopping_rule_validation():
    with pytest.raises(ValueError):
        StoppingRule("nonsense", 1e-3)
    with pytest.raises(ValueError):
        StoppingRule("relative-objective", 0.0)


def test_solver_result_trace_bound():
    with pytest.raises(ValueError):
        SolverResult(np.zeros(2), 1, 0.0, True, trace=[None] * 3)


def test_check_stop_rules():
    hist = [StopRecord(np.zeros(2), 1.0), StopRecord(np.zeros(2), 1.0)]
    assert model.check_stop(hist, StoppingRule("relative-objective", 1e-12))
    x = np.array([1.0, 2.0])
    assert model.check_stop([StopRecord(x, 3.0), StopRecord(x.copy(), 2.9)],
                            StoppingRule("relative-estimate", 1e-9))
    gt = np.array([1.0, 0.0])
    one = [StopRecord(gt + np.array([1e-2, 0.0]), 1.0)]
    assert not model.check_stop(one, StoppingRule("ground-truth-distance", 1e-3), gt)
    assert model.check_stop(one, StoppingRule("ground-truth-distance", 2e-2), gt)
    with pytest.raises(ValueError):
        model.check_stop(one, StoppingRule("ground-truth-distance", 1e-3))
    with pytest.raises(ValueError):
        model.check_stop(one, StoppingRule("relative-objective", 1e-3))
    k = [StopRecord(np.zeros(2), 1.0, kkt=1e-7)]
    assert model.check_stop(k, StoppingRule("kkt-residual", 1e-6))
    assert not model.check_stop(k, StoppingRule("kkt-residual", 1e-8))
    with pytest.raises(ValueError):
        model.check_stop([], StoppingRule("kkt-residual", 1e-6))


def test_stop_wanted_needs_history():
    P = ProblemInstance(np.eye(2), np.ones(2))
    cfg = SolverConfig(stopping=StoppingRule("relative-objective", 1e-3))
    assert not model.stop_wanted(cfg, [StopRecord(np.zeros(2), 1.0)], P)
    assert model.stop_wanted(cfg, [StopRecord(np.zeros(2), 1.0)] * 2, P)
    assert not model.stop_wanted(SolverConfig(), [StopRecord(np.zeros(2), 1.0)] * 2, P)


def test_kkt_from_correlation_cases():
    lam = 0.5
    # zero vector: violation is max|c| - lam, floored at 0
    assert model.kkt_from_correlation(np.zeros(3), np.array([0.2, -0.4, 0.1]), lam) == 0.0
    assert model.kkt_from_correlation(np.zeros(3), np.array([0.2, -0.9, 0.1]), lam) == pytest.approx(0.4)
    # on-support entries must carry c = lam sign(x)
    x = np.array([1.0, 0.0, -2.0])
    c = np.array([0.5, 0.3, -0.5])
    assert model.kkt_from_correlation(x, c, lam) == 0.0
    assert model.kkt_from_correlation(x, c + np.array([0.0, 0.0, 0.25]), lam) == pytest.approx(0.25)


def test_support_size_and_relative_error():
    assert model.support_size(np.zeros(0)) == 0
    assert model.support_size(np.array([1.0, 1e-11, 0.0, -3.0])) == 2
    assert model.support_size(np.array([1e-9, 2e-11])) == 1  # floor of max(max|x|, 1)
    assert model.relative_error(np.array([1.0, 1.0]), np.array([1.0, 0.0])) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        model.relative_error(np.ones(2), np.zeros(2))


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """Every compute entry point refuses to run without the B200 path."""
    from paper_1007_3753_b200 import numerics
    from paper_1007_3753_b200.exceptions import DeviceError
    from paper_1007_3753_b200.shrinkage import fista_solve
    with pytest.raises(DeviceError):
        numerics.soft_threshold(np.array([1.0, -2.0]), 0.5)
    with pytest.raises(DeviceError):
        fista_solve(ProblemInstance(np.eye(2), np.ones(2)), SolverConfig(tol=1e-6))
    with pytest.raises(DeviceError):
        model.objective(np.zeros(2), ProblemInstance(np.eye(2), np.ones(2)), 0.1)


def test_alm_state_validation():
    from paper_1007_3753_b200.alm import AlmState, DalmState
    AlmState(np.zeros(2), np.zeros(1), 1.0, 2.0, 3.0)
    with pytest.raises(ValueError):
        AlmState(np.zeros(2), np.zeros(1), 0.0, 2.0, 3.0)
    with pytest.raises(ValueError):
        AlmState(np.zeros(2), np.zeros(1), 1.0, 1.0, 3.0)
    DalmState(np.zeros(2), np.zeros(1), np.array([1.0, -1.0]), 1.0, None)
    with pytest.raises(ValueError):
        DalmState(np.zeros(2), np.zeros(1), np.array([1.1, 0.0]), 1.0, None)
    with pytest.raises(ValueError):
        DalmState(np.zeros(2), np.zeros(1), np.zeros(2), 0.0, None)
