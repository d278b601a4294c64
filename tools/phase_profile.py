"""Per-phase device time of the FISTA persistent kernel (diagnostics).

    python tools/phase_profile.py [--dtype float64] [--d 1024 --n 4096]
Prints mean-over-CTAs ns per iteration for each phase mark in csrc/fista.cu.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

NAMES = ["reduce12+pub", "gemv", "barrierA", "gath+slice", "q+pub", "barrierB+fin", "decide",
         "issue+gemv_t", "kkt+y+prox", "retry prox", "-"]


def main():
    import torch
    from paper_1007_3753_b200 import device as dv, synth
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig, StoppingRule
    from paper_1007_3753_b200.shrinkage import FistaPlan
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="float64")
    ap.add_argument("--d", type=int, default=1024)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--blocks", type=int, default=0, help="persistent grid size (0: one CTA per SM)")
    args = ap.parse_args()
    P = synth.make_problem(synth.Workload("p", args.d, args.n, max(1, args.n // 32), 0, 0.01))

    D = dv.DeviceDictionary(P.A, dtype=args.dtype)
    Pd = ProblemInstance.__new__(ProblemInstance)
    Pd.A, Pd.b, Pd.ground_truth = D, P.b, None
    plan = FistaPlan(Pd, SolverConfig(tol=1e-6, stopping=StoppingRule("relative-estimate", 1e-6),
                                      options={"dtype": args.dtype}))
    plan.launch()
    torch.cuda.synchronize()
    prof = torch.zeros(148 * 16, dtype=torch.int64, device=D.device)
    io = plan.bufs.io(0, blocks=args.blocks)
    io.phase_ns = prof.data_ptr()
    plan.bufs.state.zero_()
    from paper_1007_3753_b200 import _lib
    _lib.check(plan._launch(io), "fista")
    torch.cuda.synchronize()
    st = plan.bufs.read_state()
    its = st.iterations
    p = prof.cpu().numpy().reshape(148, 16)
    used = p[p.sum(axis=1) > 0]
    print("iterations", its, "blocks", used.shape[0])
    tot = 0
    for k, nm in enumerate(NAMES):
        mean = used[:, k].mean() / its
        tot += mean
        print("%-12s mean %8.0f ns  block0 %8.0f ns  max %8.0f" % (nm, mean, used[0, k] / its,
                                                                  used[:, k].max() / its))
    print("sum per iteration %.0f ns" % tot)


if __name__ == "__main__":
    main()
