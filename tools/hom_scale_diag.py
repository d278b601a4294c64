"""Config-5 Homotopy at scale: batched vs single-instance GPU vs the oracle vs
the reference golden (tests/golden/cfg5_scale.npz) per sampled instance."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1007_3753_b200 import device, synth  # noqa: E402
from paper_1007_3753_b200.batched import homotopy_solve_batch  # noqa: E402
from paper_1007_3753_b200.homotopy import solve_path  # noqa: E402
from paper_1007_3753_b200.model import SolverConfig  # noqa: E402

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cfg5_scale.npz"))
A, _, Bmat = synth.cfg5_batch(1024)
idx = [int(j) for j in g["idx"] if j < 1024]
for i, j in enumerate(g["idx"]):
    if j < 1024:
        Bmat[:, j] = g["b"][i]
D = device.DeviceDictionary(A)
res = homotopy_solve_batch(D, np.ascontiguousarray(Bmat), 1e-3, SolverConfig(max_iter=5000), with_trace=True)
rel = lambda x, r: float(np.linalg.norm(x - r) / np.linalg.norm(r))  # noqa: E731
for i, j in enumerate(g["idx"]):
    if j >= 1024:
        continue
    ref = g["homotopy_x"][i]
    rb = res.result(j)
    single, lam = solve_path(D, Bmat[:, j], 1e-3, SolverConfig(max_iter=5000))
    o, olam = oracle.homotopy(A, Bmat[:, j], 1e-3)
    tr_b = np.array([tuple(t) for t in rb.trace])
    tr_o = np.array(o.trace)
    first = -1
    if i < 4:
        tg = g["homotopy_trace_%d" % i]
        n = min(len(tg), len(tr_b))
        bad = np.nonzero(np.abs(tr_b[:n, 3] - tg[:n, 3]) > 0)[0]
        first = int(bad[0]) if bad.size else -1
    print(json.dumps(dict(j=j, it_ref=int(g["homotopy_iterations"][i]), it_batch=rb.iterations,
                          it_single=single.iterations, it_oracle=o.iterations,
                          err_batch=rel(rb.x_star, ref), err_single=rel(single.x_star, ref),
                          err_oracle=rel(o.x, ref), batch_vs_oracle=rel(rb.x_star, o.x),
                          first_support_diff_vs_ref=first, notes=rb.notes)), flush=True)
