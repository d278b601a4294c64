"""One batched-Homotopy solve at config-5 shape (profiling driver)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200 import device as dv
    from paper_1007_3753_b200.batched import homotopy_solve_batch
    from paper_1007_3753_b200.model import SolverConfig
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    A5 = synth.gen_gaussian_dict(512, 2048, 5)
    rng = np.random.default_rng(55)
    X = np.zeros((2048, B))
    for j in range(B):
        kk = int(rng.integers(16, 257))
        X[rng.choice(2048, kk, replace=False), j] = rng.standard_normal(kk)
    D = dv.DeviceDictionary(A5)
    Bm = A5 @ X
    homotopy_solve_batch(D, np.ascontiguousarray(Bm[:, :16]), 1e-3, SolverConfig())
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = homotopy_solve_batch(D, Bm, 1e-3, SolverConfig())
    e.record()
    torch.cuda.synchronize()
    print("B=%d %.1f ms %.0f solves/s mean breakpoints %.1f" % (B, s.elapsed_time(e), B / s.elapsed_time(e) * 1e3,
                                                               r.iterations.mean()))


if __name__ == "__main__":
    main()
