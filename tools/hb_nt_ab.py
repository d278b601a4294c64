"""Batched Homotopy (config 5) time per batch for the threads-per-instance
choice in ELL1_HB_NT (diagnostics; run once per setting).

    ELL1_HB_NT=128 python tools/hb_nt_ab.py 1024
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200 import device as dv
    from paper_1007_3753_b200.batched import homotopy_solve_batch
    from paper_1007_3753_b200.model import SolverConfig
    for B in [int(v) for v in sys.argv[1:]] or [1024]:
        A, _, Bmat = synth.cfg5_batch(B)
        D = dv.DeviceDictionary(A)
        homotopy_solve_batch(D, Bmat[:, :16], 1e-3, SolverConfig(max_iter=5000))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = homotopy_solve_batch(D, Bmat, 1e-3, SolverConfig(max_iter=5000))
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        print("NT=%s B=%d %.1f ms  %.0f solves/s  mean its %.2f  sum|x| %.12e" % (
            os.environ.get("ELL1_HB_NT", "auto"), B, 1e3 * t, B / t, r.iterations.mean(), np.abs(r.x).sum()))


if __name__ == "__main__":
    main()
