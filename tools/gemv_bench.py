"""Time the shard primitives ell1_gemv / ell1_gemv_t alone (diagnostics).

    python tools/gemv_bench.py [--lib path/to/libell1b200.so]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--full", action="store_true", help="only the config-4 single-GPU shape (64 GiB fp32)")
    args = ap.parse_args()
    from paper_1007_3753_b200 import _lib
    import torch
    from paper_1007_3753_b200 import device as dv
    if args.lib:
        L = ctypes.CDLL(os.path.abspath(args.lib))
        for name in ("ell1_gemv_workspace", "ell1_gemv", "ell1_gemv_t"):
            fn = getattr(L, name)
            fn.restype, fn.argtypes = _lib._SIGS[name]
    else:
        L = _lib.lib()
    dev = torch.device("cuda", 0)
    shapes = [(65536, 32768, torch.float32), (16384, 65536, torch.float32), (4096, 131072, torch.float32),
              (1024, 262144, torch.float32), (16384, 32768, torch.float64)]
    if args.full:
        shapes = [(65536, 262144, torch.float32)]
    for (d, n, dt) in shapes:
        g = torch.Generator(device=dev)
        g.manual_seed(1)
        st = torch.empty(n, d, device=dev, dtype=dt)
        for c0 in range(0, n, 8192):                    # chunked: no 2x-size temporaries at 64 GiB
            st[c0:c0 + 8192].normal_(generator=g)
        D = dv.DeviceDictionary.wrap(st, d)
        v = D.view()
        wsb = L.ell1_gemv_workspace(ctypes.byref(v))
        ws = dv.alloc_bytes(wsb, dev)
        x = torch.randn(n, dtype=torch.float64, device=dev)
        r = torch.randn(D.ld, dtype=torch.float64, device=dev)
        y = torch.zeros(D.ld, dtype=torch.float64, device=dev)
        gg = torch.zeros(n, dtype=torch.float64, device=dev)
        s = dv.stream_ptr(dev)
        for _ in range(3):
            L.ell1_gemv(ctypes.byref(v), dv.ptr(x), dv.ptr(y), dv.ptr(ws), wsb, s)
            L.ell1_gemv_t(ctypes.byref(v), dv.ptr(r), dv.ptr(gg), dv.ptr(ws), wsb, s)
        torch.cuda.synchronize()
        res = []
        for fn, a, b in ((L.ell1_gemv, x, y), (L.ell1_gemv_t, r, gg)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                fn(ctypes.byref(v), dv.ptr(a), dv.ptr(b), dv.ptr(ws), wsb, s)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 5e3
            res.append(st.numel() * st.element_size() / t / 1e9)
        print("d=%6d n=%7d %s  gemv %7.0f GB/s  gemv_t %7.0f GB/s" % (d, n, str(dt)[6:], res[0], res[1]))
        del st, D, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
