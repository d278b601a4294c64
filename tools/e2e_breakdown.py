"""Where the end-to-end fista_solve time goes (host A/b -> x) at config 2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1007_3753_b200 import device as dv, synth
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig, StoppingRule
    from paper_1007_3753_b200.shrinkage import fista_solve
    P = synth.make_problem(synth.CFG2)
    pin_A = torch.from_numpy(P.A).pin_memory()
    pin_b = torch.from_numpy(P.b).pin_memory()
    Ph = ProblemInstance(pin_A.numpy(), pin_b.numpy())
    cfg = SolverConfig(lam=None, tol=1e-6, stopping=StoppingRule("relative-estimate", 1e-6))
    for _ in range(3):
        fista_solve(Ph, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    N = 20
    for _ in range(N):
        fista_solve(Ph, cfg)
    torch.cuda.synchronize()
    print("e2e ms/solve %.3f" % ((time.perf_counter() - t0) / N * 1e3))
    # pieces
    dev = torch.device("cuda", 0)
    ts = {}
    def tim(name, fn, reps=20):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        ts[name] = (time.perf_counter() - t) / reps * 1e3
    tim("h2d A (pinned)", lambda: torch.from_numpy(Ph.A).to(dev, non_blocking=False))
    tim("DeviceDictionary(A)", lambda: dv.DeviceDictionary(Ph.A))
    D = dv.DeviceDictionary(Ph.A)
    Pd = ProblemInstance.__new__(ProblemInstance)
    Pd.A, Pd.b, Pd.ground_truth, Pd.noise_sigma = D, Ph.b, None, None
    tim("fista_solve (A resident)", lambda: fista_solve(Pd, cfg))
    from paper_1007_3753_b200.shrinkage import FistaPlan
    plan = FistaPlan(Pd, cfg)
    def launch_only():
        plan.launch()
    tim("FistaPlan.launch (kernel only)", launch_only)
    for k, v in ts.items():
        print("%-32s %.3f ms" % (k, v))


if __name__ == "__main__":
    main()
