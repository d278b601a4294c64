"""Per-phase device time of the single-instance Homotopy kernel at config 2
(diagnostics): CTA 0 (which runs the factor work) and the mean over CTAs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
NAMES = ["sgn+bar", "direction (CTA0 trsv)", "v=A_I d_I + gather", "A^T v + steps + argmin",
         "event + x", "delete", "append", "residual + corr + trace"]


def main():
    import numpy as np
    import torch
    from paper_1007_3753_b200 import _lib, device as dv, synth
    from paper_1007_3753_b200._runner import Buffers, Prepared, byref
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig
    P = synth.make_problem(synth.CFG2)
    lam = 1e-2 * float(np.max(np.abs(P.A.T @ P.b)))
    cfg = SolverConfig(lam=None, tol=1.0, max_iter=5000)
    prep = Prepared(ProblemInstance(P.A, P.b), cfg)
    L = _lib.lib()
    wsb = L.ell1_homotopy_workspace(byref(prep.view), 0)
    bufs = Buffers(prep, wsb, cfg.max_iter + 2)
    out = _lib.HomOut()
    cb = torch.zeros(prep.n, dtype=torch.float64, device=prep.dev)
    out.c = cb.data_ptr()
    prof = torch.zeros(148 * 16, dtype=torch.int64, device=prep.dev)
    io = bufs.io(0)
    io.phase_ns = prof.data_ptr()
    _lib.check(L.ell1_homotopy(byref(prep.view), dv.ptr(prep.b), lam, cfg.max_iter, byref(out), byref(io),
                               prep.stream), "homotopy")
    torch.cuda.synchronize()
    st = bufs.read_state()
    its = max(st.iterations, 1)
    p = prof.cpu().numpy().reshape(148, 16)
    used = p[p.sum(axis=1) > 0]
    print("breakpoints", st.iterations, "blocks", used.shape[0])
    t0 = tm = 0
    for k, nm in enumerate(NAMES):
        print("%-28s CTA0 %8.0f ns   mean %8.0f ns" % (nm, used[0, k] / its, used[:, k].mean() / its))
        t0 += used[0, k] / its
        tm += used[:, k].mean() / its
    print("sum per breakpoint: CTA0 %.0f ns, mean %.0f ns" % (t0, tm))


if __name__ == "__main__":
    main()
