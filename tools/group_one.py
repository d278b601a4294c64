"""One FISTA group launch (diagnostics / ncu target): 148 trials of d x n."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1007_3753_b200.group import TrialGroup            # noqa: E402
from paper_1007_3753_b200.model import SolverConfig          # noqa: E402
from paper_1007_3753_b200.synth import GenSpec, make_instance    # noqa: E402

d, n = int(sys.argv[1]), int(sys.argv[2])
name = sys.argv[3] if len(sys.argv) > 3 else "fista"
probs = [make_instance(GenSpec(n=n, d=d, k=5, seed=s)) for s in range(148)]
grp = TrialGroup(probs)
lams = 1e-4 * grp.correlation_max()
cfg = SolverConfig(tol=1e-30, max_iter=200)
for _ in range(2):
    grp.solve(name, cfg, lams=lams)
torch.cuda.synchronize()
print("ok")
