"""Name-based dispatch used by the reference's callers (ell1.bench.solve_named,
bench.py:31-62): one problem to a solver family by name, "gp" = "gpsr"."""

from paper_1007_3753_b200.alm import dalm_solve, palm_solve
from paper_1007_3753_b200.gradient_projection import gpsr_solve, tnipm_solve
from paper_1007_3753_b200.homotopy import homotopy_solve
from paper_1007_3753_b200.pdipa import pdipa_solve
from paper_1007_3753_b200.shrinkage import fista_solve, ist_solve

SOLVER_NAMES = ("pdipa", "homotopy", "gpsr", "tnipm", "ist", "fista", "palm", "dalm")


def solve_named(name, P, config):
    """Dispatch one problem to a solver family by name ("gp" = "gpsr")."""
    if name == "gp":
        name = "gpsr"
    if name == "pdipa":
        return pdipa_solve(P, config)
    if name == "homotopy":
        return homotopy_solve(P, config.resolved_lambda(P), config)
    if name == "gpsr":
        return gpsr_solve(P, config.resolved_lambda(P), config)
    if name == "tnipm":
        return tnipm_solve(P, config.resolved_lambda(P), config)
    if name == "ist":
        return ist_solve(P, None, config)
    if name == "fista":
        return fista_solve(P, config)
    if name == "palm":
        return palm_solve(P, config)
    if name == "dalm":
        return dalm_solve(P, config)
    raise ValueError("unknown solver %r (choose from %s)" % (name, ", ".join(SOLVER_NAMES)))
