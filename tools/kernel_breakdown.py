"""Per-kernel device time of the batched paths via torch.profiler (CUPTI).

    python tools/kernel_breakdown.py [--B 256]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def table(prof, title, top=12):
    from collections import defaultdict
    agg = defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type.name == "CUDA" or getattr(e, "device_type", None) is not None and "CUDA" in str(e.device_type):
            a = agg[e.name[:70]]
            a[0] += 1
            a[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    tot = sum(v[1] for v in agg.values())
    print("== %s: total kernel time %.1f ms" % (title, tot / 1e3))
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print("  %6.1f%% %9.2f ms  n=%6d  %s" % (100 * t / max(tot, 1e-9), t / 1e3, n, k))


def main():
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200 import device as dv
    from paper_1007_3753_b200.batched import (dalm_solve_batch, fista_solve_batch, homotopy_solve_batch,
                                              src_classify)
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    from paper_1007_3753_b200.robust import ExtendedDictionary
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=256)
    ap.add_argument("--math", default=None, help="ELL1_BLAS_MATH override for fp32 GEMMs")
    args = ap.parse_args()
    B = args.B
    # config 3
    A, lab = synth.cab_dictionary(d=1024, classes=38, per_class=32, subspace=9, seed=0)
    Bq, truth = synth.cab_queries(A, lab, B, fraction=0.2, seed=1)
    cfg = SolverConfig(tol=1e-4, max_iter=2000, options={"dtype": "float32"})
    ext = ExtendedDictionary(A, 1.0, dtype="float32")
    src_classify(ext, lab, np.ascontiguousarray(Bq.T[:, :8]), cfg)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        labels, _, res = src_classify(ext, lab, np.ascontiguousarray(Bq.T), cfg)
        torch.cuda.synchronize()
    table(prof, "cfg3 SRC batched DALM fp32 B=%d (mean its %.0f, acc %.3f)" % (
        B, res.iterations.mean(), float(np.mean(labels == truth))))
    # config 5
    d, n = 512, 2048
    A5 = synth.gen_gaussian_dict(d, n, 5)
    rng = np.random.default_rng(55)
    X = np.zeros((n, B))
    for j in range(B):
        kk = int(rng.integers(16, 257))
        X[rng.choice(n, kk, replace=False), j] = rng.standard_normal(kk)
    Bm = A5 @ X
    D = dv.DeviceDictionary(A5)
    rel = StoppingRule("relative-estimate", 1e-6)
    for name, fn in (("fista", lambda: fista_solve_batch(D, Bm, SolverConfig(lam=1e-3, tol=1e-6, stopping=rel))),
                     ("dalm", lambda: dalm_solve_batch(D, Bm, SolverConfig(tol=1e-6, stopping=rel))),
                     ("homotopy", lambda: homotopy_solve_batch(D, Bm, 1e-3, SolverConfig()))):
        fn()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            r = fn()
            torch.cuda.synchronize()
        table(prof, "cfg5 %s fp64 B=%d (mean its %.0f)" % (name, B, r.iterations.mean()))


if __name__ == "__main__":
    main()
