"""Experiment-harness host logic (no GPU): generators pinned to the
reference's (golden fixtures made by tests/golden/make_harness_golden.py),
result-record validation, contour interpolation and the CSV writers."""

import os

import numpy as np
import pytest

from paper_1007_3753_b200 import harness, synth

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "harness_ref.npz"))


def test_generators_match_reference():
    A, labels = synth.gen_bouquet_dict(20, 30, 5, 0.6, 3)
    np.testing.assert_array_equal(A, GOLD["bouquet_A"])
    np.testing.assert_array_equal(labels, GOLD["bouquet_labels"])
    P = synth.make_instance(synth.GenSpec(n=30, d=15, k=3, seed=5, noise_sigma=0.02))
    np.testing.assert_array_equal(P.A, GOLD["instance_A"])
    np.testing.assert_array_equal(P.b, GOLD["instance_b"])
    np.testing.assert_array_equal(P.ground_truth, GOLD["instance_x0"])
    with pytest.raises(ValueError):
        synth.GenSpec(n=3, d=2, k=4, seed=0)
    with pytest.raises(ValueError):
        synth.gen_bouquet_dict(4, 6, 2, 1.0, 0)


def test_record_validation():
    with pytest.raises(ValueError):
        harness.PhaseGrid(10, (0.1, 0.1), (0.5,), np.zeros((2, 1)), 1, 0, 1e-3)
    with pytest.raises(ValueError):
        harness.PhaseGrid(10, (0.1,), (0.5,), np.full((1, 1), 1.5), 1, 0, 1e-3)
    with pytest.raises(ValueError):
        harness.SweepResult("d", (1, 2), ("fista",), 1, np.zeros((1, 3)))
    with pytest.raises(ValueError):
        harness.run_phase_grid("fista", 10, (0.1,), (0.5,), 0)
    with pytest.raises(ValueError):
        harness.run_noise_sweep(("fista",), "vary-x", {"n": 10}, 1)


def test_contour_and_csv(tmp_path):
    g = harness.PhaseGrid(10, (0.1, 0.2, 0.3), (0.4, 0.8),
                          np.array([[1.0, 1.0], [0.5, 1.0], [0.0, 0.75]]), 4, 0, 1e-3)
    pts = harness.interpolate_success_contour(g, 0.5)
    assert len(pts) == 1 and pts[0] == (0.4, pytest.approx(0.2))     # the 0.8 column never drops below 0.5
    with pytest.raises(ValueError):
        harness.interpolate_success_contour(g, 1.0)
    p = harness.phase_grid_to_csv(g, str(tmp_path / "g.csv"))
    rows = open(p).read().splitlines()
    assert rows[0] == "rho,delta,success_rate" and rows[1] == "0.10000000000000001,0.40000000000000002,1"
    s = harness.SweepResult("d", (20, 30), ("fista", "ist"), 2, np.ones((2, 2)),
                            mean_rel_error=np.zeros((2, 2)), mean_iterations=np.full((2, 2), 3.0))
    rows = open(harness.sweep_to_csv(s, str(tmp_path / "s.csv"))).read().splitlines()
    assert rows[0] == "d,solver,mean_time_seconds,mean_rel_error,mean_iterations"
    assert rows[1] == "20,fista,1,0,3" and len(rows) == 5
