"""One config-3 SRC batch (1024 queries, batched DALM fp32 on [A I]) — profiling driver."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200.batched import src_classify
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.robust import ExtendedDictionary
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    A, lab = synth.cab_dictionary(d=1024, classes=38, per_class=32, subspace=9, seed=0)
    Bq, truth = synth.cab_queries(A, lab, B, fraction=0.2, seed=1)
    cfg = SolverConfig(tol=1e-4, max_iter=2000, options={"dtype": "float32"})
    ext = ExtendedDictionary(A, 1.0, dtype="float32")
    src_classify(ext, lab, np.ascontiguousarray(Bq.T[:, :8]), cfg)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    torch.cuda.nvtx.range_push("main")
    labels, _, res = src_classify(ext, lab, np.ascontiguousarray(Bq.T), cfg)
    torch.cuda.nvtx.range_pop()
    e.record()
    torch.cuda.synchronize()
    print("B=%d %.1f ms  %.0f queries/s  mean its %.1f  acc %.4f" % (
        B, s.elapsed_time(e), B / s.elapsed_time(e) * 1e3, res.iterations.mean(), float(np.mean(labels == truth))))


if __name__ == "__main__":
    main()
