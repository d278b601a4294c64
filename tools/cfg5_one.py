"""One config-5 batched FISTA fp64 solve (B instances sharing A 512 x 2048) — profiling driver."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200 import device as dv
    from paper_1007_3753_b200.batched import fista_solve_batch
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    A, _, Bmat = synth.cfg5_batch(B)
    D = dv.DeviceDictionary(A, dtype="float64")
    cfg = SolverConfig(lam=1e-3, tol=1e-6, max_iter=5000, stopping=StoppingRule("relative-estimate", 1e-6))
    fista_solve_batch(D, Bmat[:, :16], cfg)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("main")
    r = fista_solve_batch(D, Bmat, cfg)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    print("B=%d mean its %.1f" % (B, r.iterations.mean()))


if __name__ == "__main__":
    main()
