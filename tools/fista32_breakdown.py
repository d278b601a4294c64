"""Per-kernel device time of the batched FISTA fp32 / fp64 path at config 5 (torch.profiler).

    python tools/fista32_breakdown.py [B] [float32|float64]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kernel_breakdown import table  # noqa: E402


def main():
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_1007_3753_b200 import device as dv, synth
    from paper_1007_3753_b200.batched import fista_solve_batch
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    dt = sys.argv[2] if len(sys.argv) > 2 else "float32"
    A, _, Bmat = synth.cfg5_batch(B)
    D = dv.DeviceDictionary(A, dtype=dt)
    cfg = SolverConfig(lam=1e-3, stopping=StoppingRule("relative-estimate", 1e-6))
    if not os.environ.get("NO_WARM"):                      # ncu captures: skip the small warm-up solve
        fista_solve_batch(D, np.ascontiguousarray(Bmat[:, :16]), cfg)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = fista_solve_batch(D, Bmat, cfg)
    e.record()
    torch.cuda.synchronize()
    print("B=%d %s: %.1f ms, %.0f solves/s, mean its %.0f max %d" % (
        B, dt, s.elapsed_time(e), B / s.elapsed_time(e) * 1e3, r.iterations.mean(), r.iterations.max()))
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = fista_solve_batch(D, Bmat, cfg)
        torch.cuda.synchronize()
    table(prof, "cfg5 fista %s B=%d" % (dt, B))


if __name__ == "__main__":
    main()
