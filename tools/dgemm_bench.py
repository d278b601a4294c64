"""ell1_gemm_f64 (own DMMA kernel) vs torch.matmul (cuBLAS DGEMM) at the
batched solvers' shapes: accuracy against an fp64 reference and time per
call (CUDA events, best of 5 after warm-up)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1007_3753_b200 import _lib  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda", 0)
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ours(ta, tb, m, n, k, A, lda, B, ldb, C, variant=None, split=-1):
    if variant is None:
        rc = L.ell1_gemm_f64(ta, tb, m, n, k, P(A), lda, P(B), ldb, P(C), m, stream)
    else:
        rc = L.ell1_gemm_f64_variant(variant, split, ta, tb, m, n, k, P(A), lda, P(B), ldb, P(C), m, stream)
    assert rc == 0, rc


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


rows = []
shapes = [("AX", 0, 0, 512, B, 2048) for B in (64, 256, 485, 1024, 2048, 8192)] + \
         [("AtR", 1, 0, 2048, B, 512) for B in (64, 256, 485, 1024, 2048, 8192)] + \
         [("GinvB", 0, 0, 1024, 1024, 1024), ("AX_cab", 0, 0, 1024, 2048, 2240),
          ("gramNT", 0, 1, 1024, 1024, 4096), ("big", 0, 0, 4096, 4096, 4096)]
for name, ta, tb, m, n, k in shapes:
    # column-major storage as row-major transposes
    A_cm = torch.randn(k if ta == 0 else m, m if ta == 0 else k, dtype=torch.float64, device=dev)  # rows = cols of A
    lda = m if ta == 0 else k
    B_cm = torch.randn(n if tb == 0 else k, k if tb == 0 else n, dtype=torch.float64, device=dev)
    ldb = k if tb == 0 else n
    C = torch.empty(n, m, dtype=torch.float64, device=dev)
    opA = A_cm.T if ta == 0 else A_cm          # (m x k) logical
    opB = B_cm.T if tb == 0 else B_cm          # (k x n) logical
    ref = opA @ opB
    ours(ta, tb, m, n, k, A_cm, lda, B_cm, ldb, C)
    torch.cuda.synchronize()
    err = float(((C.T - ref).abs().max() / (opA.abs() @ opB.abs()).max()).item())
    t_o = timeit(lambda: ours(ta, tb, m, n, k, A_cm, lda, B_cm, ldb, C))
    t_c = timeit(lambda: torch.matmul(opA, opB))
    fl = 2.0 * m * n * k
    sweep = {}
    if os.environ.get("SWEEP", "1") == "1":
        for v in range(5):
            for sp in (1, 2, 4, 8):
                try:
                    tv = timeit(lambda: ours(ta, tb, m, n, k, A_cm, lda, B_cm, ldb, C, v, sp), reps=3)
                    sweep["v%d_s%d" % (v, sp)] = round(fl / tv / 1e12, 2)
                except AssertionError:
                    pass
    best = max(sweep.items(), key=lambda kv: kv[1]) if sweep else None
    rows.append(dict(name=name, m=m, n=n, k=k, err=err, ours_us=1e6 * t_o, cublas_us=1e6 * t_c,
                     ours_tflops=fl / t_o / 1e12, cublas_tflops=fl / t_c / 1e12, best=best, sweep=sweep))
    print(json.dumps(rows[-1]), flush=True)
