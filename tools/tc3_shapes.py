"""tcgen05 3xTF32 GEMM time at the config-3 shapes (ell1_gemm_f32)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1007_3753_b200 import _lib  # noqa: E402

L = _lib.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for name, tr, M, N, K in (("A[U|x] 2B", 0, 1024, 2048, 1216), ("A U  B", 0, 1024, 1024, 1216),
                          ("A^T Y", 1, 1216, 1024, 1024), ("[M|G^-1] V", 0, 1024, 1024, 2240),
                          ("A Z", 0, 1024, 1024, 1216), ("G Y", 0, 1024, 1024, 1024)):
    A = torch.randn((K, M) if tr else (M * 0 + K, M), dtype=torch.float32, device="cuda") if tr else \
        torch.randn(K, M, dtype=torch.float32, device="cuda")          # column-major M x K (lda = M) or K x M
    lda = K if tr else M
    if tr:
        A = torch.randn(M, K, dtype=torch.float32, device="cuda")       # column-major K x M: M columns of K
    B = torch.randn(N, K, dtype=torch.float32, device="cuda")           # column-major K x N
    C = torch.empty(N, M, dtype=torch.float32, device="cuda")
    wsb = L.ell1_gemm_f32_workspace(tr, M, K)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    f = lambda: L.ell1_gemm_f32(tr, M, N, K, P(A), lda, P(B), K, P(C), M, P(ws), wsb, st)  # noqa: E731
    f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    print("%-12s M=%d N=%d K=%d  %.1f us  %.0f TF/s (x3 tf32)" % (name, M, N, K, best * 1e3,
                                                                3 * 2 * M * N * K / best / 1e9), flush=True)
