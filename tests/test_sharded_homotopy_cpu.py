"""Column-sharded Homotopy control loop on CPU: the
host driver of paper_1007_3753_b200/sharded_homotopy.py over numpy shard ops
(tests/shard_numpy_ops.py), at world size 1 and 2 over gloo, against the
reference's golden paths — same breakpoints, trace, lambda and x."""

import os

import numpy as np
import pytest

from tests.gpu_util import assert_parity, case_inputs
from tests.golden.cases import resolve_lambda

CASES = ["homotopy_small_1300", "homotopy_small_1301", "cfg5_homotopy_k16"]


def _solve(cid, rank, world):
    from types import SimpleNamespace
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.sharded import column_range
    from paper_1007_3753_b200.sharded_homotopy import sharded_solve_path
    from tests.shard_numpy_ops import NumpyHomShardOps
    case, A, b, gt, gold = case_inputs(cid)
    lam = resolve_lambda(case["cfg"], A, b)
    target = lam if lam is not None else 1e-2 * float(np.max(np.abs(A.T @ b)))
    c0, c1 = column_range(A.shape[1], rank, world)
    shard = SimpleNamespace(c0=c0, c1=c1, d=A.shape[0], n=A.shape[1])
    P = SimpleNamespace(A=shard, b=b)
    res, lam_r = sharded_solve_path(P, target, SolverConfig(max_iter=case["cfg"].get("max_iter", 5000)),
                                    ops=NumpyHomShardOps(A[:, c0:c1], A.shape[1]))
    return res, lam_r, gold


@pytest.mark.parametrize("cid", CASES)
def test_sharded_homotopy_world1_matches_golden(cid):
    res, lam, gold = _solve(cid, 0, 1)
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-9)


def _worker(rank, world, port, out_dir, cids):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for cid in cids:
            res, lam, _ = _solve(cid, rank, world)
            tr = np.array([tuple(t) for t in res.trace], dtype=np.float64).reshape(-1, 4)
            np.savez(os.path.join(out_dir, "%s_r%d.npz" % (cid, rank)), x=res.x_star,
                     iterations=res.iterations, converged=res.converged, trace=tr, lam=lam)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_homotopy_gloo_matches_golden(tmp_path, world):
    import socket
    import torch.multiprocessing as mp
    from tests.golden.run_oracle import load_golden
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(world, port, str(tmp_path), CASES), nprocs=world, join=True)
    for cid in CASES:
        gold = load_golden(cid)
        outs = [np.load(os.path.join(tmp_path, "%s_r%d.npz" % (cid, r))) for r in range(world)]
        for o in outs:
            assert_parity(o["x"], int(o["iterations"]), bool(o["converged"]),
                          [tuple(t) for t in o["trace"]], gold, 1e-9)
            np.testing.assert_array_equal(o["x"], outs[0]["x"])
