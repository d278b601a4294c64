"""A/B of the config-4 GEMV paths: d = 65536 (bulk-copy stream kernel) vs
d = 65504 (engine panel kernel; d % 32 != 0 keeps it off the stream path),
fp32, n = 32768 (the 8-way shard), CUDA events, best of 5."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1007_3753_b200 import _lib, device  # noqa: E402

L = _lib.lib()
for d in (65536, 65504, 65536, 65504):
    n = 32768
    ld = (d + 31) // 32 * 32
    st = torch.randn(n, ld, device="cuda", dtype=torch.float32)
    D = device.DeviceDictionary.wrap(st, d)
    v = D.view()
    wsb = L.ell1_gemv_workspace(ctypes.byref(v))
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.zeros(ld, dtype=torch.float64, device="cuda")
    r = torch.randn(ld, dtype=torch.float64, device="cuda")
    g = torch.zeros(n, dtype=torch.float64, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    best = {}
    for name, fn in (("gemv", lambda: L.ell1_gemv(ctypes.byref(v), P(x), P(y), P(ws), wsb, sp)),
                     ("gemv_t", lambda: L.ell1_gemv_t(ctypes.byref(v), P(r), P(g), P(ws), wsb, sp))):
        fn()
        torch.cuda.synchronize()
        b = 1e9
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            b = min(b, s.elapsed_time(e) / 1e3)
        best[name] = round(d * n * 4 / b / 1e9, 1)
    print(d, best, flush=True)
    del st, D, ws
    torch.cuda.empty_cache()
