"""Per-kernel device time of one PDIPA solve at config 2 (torch.profiler)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kernel_breakdown import table  # noqa: E402


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_1007_3753_b200 import device as dv, synth
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig
    from paper_1007_3753_b200.pdipa import pdipa_solve
    P = synth.make_problem(synth.CFG2)
    D = dv.DeviceDictionary(P.A)
    Pd = ProblemInstance.__new__(ProblemInstance)
    Pd.A, Pd.b, Pd.ground_truth, Pd.noise_sigma = D, P.b, P.ground_truth, P.noise_sigma
    cfg = SolverConfig(tol=1e-6)
    pdipa_solve(Pd, cfg)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = pdipa_solve(Pd, cfg)
    e.record()
    torch.cuda.synchronize()
    print("pdipa cfg2: %.1f ms, %d iterations, %.0f us/iteration" % (
        s.elapsed_time(e), r.iterations, 1e3 * s.elapsed_time(e) / max(r.iterations, 1)))
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        pdipa_solve(Pd, cfg)
        torch.cuda.synchronize()
    table(prof, "pdipa cfg2", top=16)


if __name__ == "__main__":
    main()
