"""Per-phase device time of the single-instance DALM kernel (diagnostics),
config 1 or 2 instance: mean over CTAs of each mark interval per iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
NAMES = ["z-step + M v, A z partials", "bar + gather y/rhs", "bar + gather", "A^T y",
         "x-step + A A^T y, A x", "barrier", "gather cert + count", "barrier", "gather + decide / refine",
         "trace/conv"]


def main():
    import torch
    from paper_1007_3753_b200 import _lib, device as dv, synth
    from paper_1007_3753_b200._runner import Buffers, Prepared, byref
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig
    w = synth.CFG1 if "cfg1" in sys.argv else synth.CFG2
    blocks = 0
    for arg in sys.argv[1:]:
        if arg.startswith("small="):                       # small=d,n,blocks (group-trial shape)
            d, n, blocks = (int(v) for v in arg[6:].split(","))
            w = synth.Workload("small", d, n, max(1, d // 10), 0, 0.0)
    P = synth.make_problem(w)
    cfg = SolverConfig(tol=1e-8, max_iter=300)
    prep = Prepared(ProblemInstance(P.A, P.b), cfg)
    D = prep.D
    MT, Gcm, _, _ = D.gram_factor(False, 0.0)
    O = _lib.DalmOpts()
    O.beta, O.y_tol, O.y_cg_step = 1.0, 1e-10, 0
    O.M, O.Ginv = MT.data_ptr(), Gcm.data_ptr()
    L = _lib.lib()
    bufs = Buffers(prep, L.ell1_dalm_workspace(byref(prep.view), 0), cfg.max_iter + 2)
    prof = torch.zeros(148 * 16, dtype=torch.int64, device=prep.dev)
    io = bufs.io(0, blocks=blocks)
    io.phase_ns = prof.data_ptr()
    _lib.check(L.ell1_dalm(byref(prep.view), dv.ptr(prep.b), byref(prep.ctrl), byref(O), byref(io),
                           prep.stream), "dalm")
    torch.cuda.synchronize()
    st = bufs.read_state()
    its = max(st.iterations, 1)
    p = prof.cpu().numpy().reshape(148, 16)
    used = p[p.sum(axis=1) > 0]
    print(w.name, "iterations", st.iterations, "blocks", used.shape[0])
    tot = 0
    for k, nm in enumerate(NAMES[:9]):
        v = used[:, k].mean() / its
        tot += v
        print("%-30s mean %8.0f ns" % (nm, v))
    print("sum per iteration %.0f ns" % tot)


if __name__ == "__main__":
    main()
