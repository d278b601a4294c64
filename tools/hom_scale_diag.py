"""Config-5 Homotopy at scale: batched (B=1024 / 8192) vs the reference golden
(tests/golden/cfg5_scale.npz) per sampled instance: iterations, x error,
objective, final KKT, first trace divergence."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1007_3753_b200 import device, synth  # noqa: E402
from paper_1007_3753_b200.batched import homotopy_solve_batch  # noqa: E402
from paper_1007_3753_b200.model import SolverConfig  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cfg5_scale.npz"))
A, _, Bmat = synth.cfg5_batch(B)
for i, j in enumerate(g["idx"]):
    if j < B:
        Bmat[:, j] = g["b"][i]
D = device.DeviceDictionary(A)
res = homotopy_solve_batch(D, np.ascontiguousarray(Bmat), 1e-3, SolverConfig(max_iter=5000), with_trace=True)
rel = lambda x, r: float(np.linalg.norm(x - r) / np.linalg.norm(r))  # noqa: E731
for i, j in enumerate(g["idx"]):
    if j >= B:
        continue
    j = int(j)
    rb = res.result(j)
    ref = g["homotopy_x"][i]
    xs = rb.x_star
    c = A.T @ (Bmat[:, j] - A @ xs)
    on = xs != 0
    kkt = max(float(np.max(np.abs(c[on] - 1e-3 * np.sign(xs[on])))) if on.any() else 0.0,
              float(np.max(np.abs(c[~on]) - 1e-3)) if (~on).any() else 0.0, 0.0)
    first = -1
    if i < 4:
        tg = g["homotopy_trace_%d" % i]
        tb = np.array([tuple(t) for t in rb.trace])
        nmin = min(len(tg), len(tb))
        bad = np.nonzero((tb[:nmin, 3] != tg[:nmin, 3]) | (np.abs(tb[:nmin, 1] - tg[:nmin, 1]) > 1e-9 * np.abs(tg[:nmin, 1])))[0]
        first = int(bad[0]) if bad.size else -1
    print(json.dumps(dict(j=j, it_ref=int(g["homotopy_iterations"][i]), it=int(rb.iterations), err=rel(xs, ref),
                          F=float(rb.trace[-1].objective), F_ref=float(g["homotopy_last_trace"][i][1]),
                          lam=float(res.lam[j]), kkt=kkt, first_diff=first, notes=list(rb.notes))), flush=True)
