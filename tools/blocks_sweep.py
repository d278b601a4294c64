"""FISTA solve time vs persistent-grid size (io.blocks) at configs 1 and 2.

    python tools/blocks_sweep.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1007_3753_b200 import _lib, device as dv, synth
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig, StoppingRule
    from paper_1007_3753_b200.shrinkage import FistaPlan
    rel = StoppingRule("relative-estimate", 1e-6)
    for name, spec, lam in (("cfg1", synth.CFG1, 1e-3), ("cfg2", synth.CFG2, None)):
        P = synth.make_problem(spec)
        D = dv.DeviceDictionary(P.A)
        Pd = ProblemInstance.__new__(ProblemInstance)
        Pd.A, Pd.b, Pd.ground_truth, Pd.noise_sigma = D, P.b, P.ground_truth, P.noise_sigma
        cfg = SolverConfig(lam=lam, tol=1e-6, stopping=rel)
        plan = FistaPlan(Pd, cfg)
        L = _lib.lib()
        from ctypes import byref
        ref = None
        for nb in (16, 24, 32, 40, 48, 64, 96, 128, 148):
            plan.ws_bytes = L.ell1_fista_workspace(byref(plan.prep.view), byref(plan.prep.ctrl), nb)
            plan.bufs = None
            plan._alloc(False)
            def run():
                plan.bufs.state.zero_()
                _lib.check(plan._launch(plan.bufs.io(0, nb)), "ell1_fista")
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            reps = 20
            s.record()
            for _ in range(reps):
                run()
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / reps
            r = plan.result()
            if ref is None:
                ref = r.x_star
            err = float(np.linalg.norm(r.x_star - ref) / np.linalg.norm(ref))
            print("%s nb=%3d  %.3f ms/solve  %d its  %.2f us/it  rel-diff %.1e" % (
                name, nb, ms, r.iterations, 1e3 * ms / r.iterations, err), flush=True)


if __name__ == "__main__":
    main()
