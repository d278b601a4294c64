"""Config-3 batched DALM (fp32, 1024 CAB queries) with and without the CUDA-graph loop."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1007_3753_b200 import synth  # noqa: E402
from paper_1007_3753_b200.batched import src_classify  # noqa: E402
from paper_1007_3753_b200.model import SolverConfig  # noqa: E402
from paper_1007_3753_b200.robust import ExtendedDictionary  # noqa: E402

A, lab = synth.cab_dictionary(d=1024, classes=38, per_class=32, subspace=9, seed=0)
Bq, truth = synth.cab_queries(A, lab, 1024, fraction=0.2, seed=1)
ext = ExtendedDictionary(A, 1.0, dtype="float32")
cfg = SolverConfig(tol=1e-4, max_iter=2000, options={"dtype": "float32"})
Bm = np.ascontiguousarray(Bq.T)
src_classify(ext, lab, Bm, cfg)
for g in ("1", "0", "1"):
    os.environ["ELL1_BATCH_GRAPH"] = g
    torch.cuda.synchronize()
    t = time.perf_counter()
    lab_, _, r = src_classify(ext, lab, Bm, cfg)
    torch.cuda.synchronize()
    print("graph", g, 1024 / (time.perf_counter() - t), r.iterations.mean(), flush=True)
