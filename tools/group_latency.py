"""Per-iteration latency of group launches vs trial shape (diagnostics):
for each (d, n), 4 x 148 identical-shape FISTA trials at fixed iterations."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1007_3753_b200 import _lib                      # noqa: E402
from paper_1007_3753_b200.group import TrialGroup           # noqa: E402
from paper_1007_3753_b200.model import SolverConfig         # noqa: E402
from paper_1007_3753_b200.synth import GenSpec, make_instance   # noqa: E402

for d, n in [(40, 200), (100, 200), (140, 200), (200, 200), (100, 400), (380, 400)]:
    probs = [make_instance(GenSpec(n=n, d=d, k=5, seed=s)) for s in range(592)]
    grp = TrialGroup(probs)
    team = int(_lib.lib().ell1_group_team(_lib.SOLVER_FISTA, ctypes.byref(grp.dicts[0])))
    lams = 1e-4 * grp.correlation_max()
    cfg = SolverConfig(tol=1e-30, max_iter=200)
    grp.solve("fista", cfg, lams=lams)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    res = grp.solve("fista", cfg, lams=lams)
    e.record()
    torch.cuda.synchronize()
    its = sum(r.iterations for r in res)
    ms = s.elapsed_time(e)
    conc = 148 // team
    print("d=%d n=%d team=%d: %.2f ms, %d trial-iterations, %.2f us/iteration per team (concurrency %d)"
          % (d, n, team, ms, its, 1e3 * ms / (its / conc), conc), flush=True)
