"""Library GEMM peaks on this GPU pool (cuBLAS via torch, 8192^3, best of 5):
the denominators of the batched solvers' tensor-pipe rooflines (only bf16 is
in MEASURED_PEAKS.json).  Run once per pool; bench.py reads the JSON so its
own launch list carries no library kernels.

    python tools/gemm_peaks.py > profiles/r02_gemm_peaks.json
"""
import json

import torch


def peak(dtype, tf32=False):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(8192, 8192, device="cuda", dtype=dtype)
    b = torch.randn(8192, 8192, device="cuda", dtype=dtype)
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        torch.cuda.synchronize()
        best = max(best, 2 * 8192 ** 3 / (s.elapsed_time(e) / 1e3) / 1e12)
    return best


print(json.dumps({"dgemm_tflops": peak(torch.float64), "sgemm_tflops": peak(torch.float32),
                  "tf32_tflops": peak(torch.float32, True), "gpu": torch.cuda.get_device_name(0),
                  "how": "torch.matmul 8192^3, best of 5, CUDA events"}))
