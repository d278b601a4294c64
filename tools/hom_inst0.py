"""Instance 0 of the config-5 batch: batched Homotopy trace tail at B=8192
against the reference's trace (where the path diverges and how)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1007_3753_b200 import device, synth  # noqa: E402
from paper_1007_3753_b200.batched import homotopy_solve_batch  # noqa: E402
from paper_1007_3753_b200.homotopy import solve_path  # noqa: E402
from paper_1007_3753_b200.model import SolverConfig  # noqa: E402

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cfg5_scale.npz"))
tg = g["homotopy_trace_0"]
for B in (int(a) for a in sys.argv[1:] or ["8192", "4096", "2048"]):
    A, _, Bmat = synth.cfg5_batch(B)
    for i, j in enumerate(g["idx"]):
        if j < B:
            Bmat[:, j] = g["b"][i]
    D = device.DeviceDictionary(A)
    res = homotopy_solve_batch(D, np.ascontiguousarray(Bmat), 1e-3, SolverConfig(max_iter=5000), with_trace=True)
    r = res.result(0)
    tb = np.array([tuple(t) for t in r.trace])
    print("B=%d it=%d lam=%.17g notes=%s" % (B, r.iterations, res.lam[0], r.notes))
    for k in range(798, min(len(tb), len(tg) + 3)):
        a = tb[k] if k < len(tb) else None
        b = tg[k] if k < len(tg) else None
        print(k, a, b)
single, lam = solve_path(device.DeviceDictionary(A), Bmat[:, 0], 1e-3, SolverConfig(max_iter=5000))
print("single-instance GPU:", single.iterations, lam, np.linalg.norm(single.x_star - g["homotopy_x"][0]) / np.linalg.norm(g["homotopy_x"][0]))
