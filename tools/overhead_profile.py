"""cProfile of fista_solve with a resident dictionary (host overhead around the kernel)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1007_3753_b200 import device as dv, synth
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig, StoppingRule
    from paper_1007_3753_b200.shrinkage import fista_solve
    P = synth.make_problem(synth.CFG2)
    D = dv.DeviceDictionary(P.A)
    Pd = ProblemInstance.__new__(ProblemInstance)
    Pd.A, Pd.b, Pd.ground_truth, Pd.noise_sigma = D, P.b, None, None
    cfg = SolverConfig(lam=None, tol=1e-6, stopping=StoppingRule("relative-estimate", 1e-6))
    for _ in range(5):
        fista_solve(Pd, cfg)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        fista_solve(Pd, cfg)
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
