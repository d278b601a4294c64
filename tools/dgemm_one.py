"""A few ell1_gemm_f64 launches at one shape (for ncu):  python tools/dgemm_one.py TA TB M N K [variant split]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1007_3753_b200 import _lib  # noqa: E402

ta, tb, m, n, k = (int(v) for v in sys.argv[1:6])
variant = int(sys.argv[6]) if len(sys.argv) > 6 else -1
split = int(sys.argv[7]) if len(sys.argv) > 7 else -1
L = _lib.lib()
dev = torch.device("cuda", 0)
A = torch.randn((k if ta == 0 else m) * (m if ta == 0 else k), dtype=torch.float64, device=dev)
B = torch.randn((n if tb == 0 else k) * (k if tb == 0 else n), dtype=torch.float64, device=dev)
C = torch.empty(n * m, dtype=torch.float64, device=dev)
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    if variant < 0:
        rc = L.ell1_gemm_f64(ta, tb, m, n, k, P(A), m if ta == 0 else k, P(B), k if tb == 0 else n, P(C), m, st)
    else:
        rc = L.ell1_gemm_f64_variant(variant, split, ta, tb, m, n, k, P(A), m if ta == 0 else k, P(B),
                                     k if tb == 0 else n, P(C), m, st)
    assert rc == 0
torch.cuda.synchronize()
print("ok")
