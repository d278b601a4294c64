"""Column-sharded FISTA control loop (BASELINE config 4) on CPU: the host
driver of paper_1007_3753_b200/sharded.py over numpy shard ops, at world size
1 in-process and 2 / 3 over torch.distributed gloo, checked against the
reference's golden outputs (tests/golden) — same iterations, trace and x."""

import os
import socket
import tempfile
from types import SimpleNamespace

import numpy as np
import pytest

from tests.gpu_util import assert_parity, case_inputs, make_config

CASES = ["fista_small_1400", "fista_small_1401", "fista_small_exactL", "fista_small_relobj",
         "fista_small_kktrule", "fista_small_gtrule", "fista_small_budget",
         "fista_small_noncont", "fista_qr", "cfg1_fista"]


def _solve(cid, rank, world):
    from paper_1007_3753_b200.sharded import column_range, sharded_fista_solve
    from tests.shard_numpy_ops import NumpyShardOps
    case, A, b, gt, gold = case_inputs(cid)
    cfg = make_config(case, A, b)
    c0, c1 = column_range(A.shape[1], rank, world)
    shard = SimpleNamespace(c0=c0, c1=c1, d=A.shape[0], n=A.shape[1])
    P = SimpleNamespace(A=shard, b=b, ground_truth=gt)
    return sharded_fista_solve(P, cfg, ops=NumpyShardOps(A[:, c0:c1], A.shape[1])), gold


@pytest.mark.parametrize("cid", CASES)
def test_sharded_world1_matches_golden(cid):
    res, gold = _solve(cid, 0, 1)
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-9)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, cids):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for cid in cids:
            res, _ = _solve(cid, rank, world)
            tr = np.array([tuple(t) for t in res.trace], dtype=np.float64).reshape(-1, 4)
            np.savez(os.path.join(out_dir, "%s_r%d.npz" % (cid, rank)), x=res.x_star,
                     iterations=res.iterations, converged=res.converged, trace=tr)
    finally:
        dist.destroy_process_group()


def _run_world(world, cids):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), tmp, cids), nprocs=world, join=True)
        out = {}
        for cid in cids:
            out[cid] = [dict(np.load(os.path.join(tmp, "%s_r%d.npz" % (cid, r))))
                        for r in range(world)]
        return out


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gloo_matches_golden(world):
    cids = ["fista_small_1400", "fista_small_exactL", "fista_small_gtrule",
            "fista_small_noncont", "cfg1_fista"]
    out = _run_world(world, cids)
    for cid in cids:
        _, _, _, _, gold = case_inputs(cid)
        r0 = out[cid][0]
        # every rank holds the same full x and took the same decisions
        for rr in out[cid][1:]:
            np.testing.assert_array_equal(rr["x"], r0["x"])
            assert int(rr["iterations"]) == int(r0["iterations"])
        trace = [tuple(t) for t in r0["trace"]]
        assert_parity(r0["x"], int(r0["iterations"]), bool(r0["converged"]), trace, gold, 1e-9)


def test_column_range_partitions():
    from paper_1007_3753_b200.sharded import column_range
    for n in (1, 7, 100, 262144):
        for world in (1, 2, 3, 8):
            spans = [column_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            sizes = [c1 - c0 for c0, c1 in spans]
            assert max(sizes) - min(sizes) <= 1
