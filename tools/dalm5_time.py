"""Config-5 batched DALM (fp64, B=1024) solves/s, twice."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1007_3753_b200 import device, synth  # noqa: E402
from paper_1007_3753_b200.batched import dalm_solve_batch  # noqa: E402
from paper_1007_3753_b200.model import SolverConfig, StoppingRule  # noqa: E402

A, _, B = synth.cfg5_batch(1024)
D = device.DeviceDictionary(A)
D.gram_factor()
cfg = SolverConfig(max_iter=5000, stopping=StoppingRule("relative-estimate", 1e-6))
dalm_solve_batch(D, B[:, :64], cfg)
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = dalm_solve_batch(D, B, cfg)
    torch.cuda.synchronize()
    print("cfg5 dalm", 1024 / (time.perf_counter() - t), r.iterations.mean(), flush=True)
