"""Oracle pin for the alignment PALM restatement (oracle.l1_oracle.align_palm,
robust.py:470-515): bit-identical to the reference's outputs on every golden
PALM case (tests/golden/make_align_golden.py)."""

import os

import numpy as np
import pytest

from oracle.l1_oracle import align_palm
from tests.golden.align_cases import CASES, align_instance

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "align_golden.npz")


@pytest.mark.parametrize("name", sorted(n for n, c in CASES.items() if c["solver"] == "palm"))
def test_align_palm_oracle_matches_reference(name):
    c = CASES[name]
    g = np.load(GOLD)
    B, b = align_instance(**c["recipe"])
    o = c.get("options", {})
    w, e = align_palm(B, b, tol=c["tol"], max_iter=c["max_iter"], mu0=o.get("mu0", 1.0), rho=o.get("rho", 2.0))
    assert np.array_equal(w, g[name + "_w"]) and np.array_equal(e, g[name + "_e"])
