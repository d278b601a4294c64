"""Instance-sharded batches over torch.distributed/gloo (world size 2 and 3):
the sharding / gather / reorder logic of paper_1007_3753_b200/distributed.py
with the oracle standing in for the per-rank GPU batch solver."""

import os
import socket
import tempfile

import numpy as np
import pytest

import oracle


def _oracle_batch(A, Bsub, config):
    """Test stand-in for batched.fista_solve_batch on one rank's share."""
    from paper_1007_3753_b200.batched import BatchResult
    xs, its, conv = [], [], []
    for j in range(Bsub.shape[1]):
        r = oracle.fista(A, Bsub[:, j], lam=config["lam"], tol=1e-6, stop=("relative-estimate", 1e-6))
        xs.append(r.x)
        its.append(r.iterations)
        conv.append(int(r.converged))
    n = A.shape[1]
    x = np.stack(xs, axis=1) if xs else np.zeros((n, 0))
    res = BatchResult(x, np.array(its, np.int32), np.array(conv, np.int32), np.zeros(len(its), np.int32), 0.0,
                      None, "homotopy")
    res.lam = np.array([float(j) for j in range(len(its))]) + 0.5
    return res


def _oracle_classify(A, labels, Bsub, config):
    B = Bsub.shape[1]
    lab = np.array([int(np.argmax(np.abs(A.T @ Bsub[:, j]))) % 3 for j in range(B)], np.int32)
    res = np.stack([np.full(3, float(j)) for j in range(B)]) if B else np.zeros((0, 3))
    return lab, res, None


def _oracle_align(Bs, bs, config):
    """Test stand-in for robust.align_palm_solve_batch on one rank's images."""
    from oracle.l1_oracle import align_palm
    ws, es = [], []
    for B, b in zip(Bs, bs):
        w, e = align_palm(B, b, tol=config["tol"])
        ws.append(w)
        es.append(e)
    m, d = Bs.shape[2], Bs.shape[1]
    return (np.stack(ws) if ws else np.zeros((0, m))), (np.stack(es) if es else np.zeros((0, d)))


def _align_problem():
    from tests.golden.align_cases import align_instance
    insts = [align_instance(seed=50 + j, d=30, m=3) for j in range(7)]
    return np.stack([B for B, _ in insts]), np.stack([b for _, b in insts])


def _problem():
    A = oracle.gaussian_dict(30, 60, 3)
    rng = np.random.default_rng(4)
    X = np.zeros((60, 7))
    for j in range(7):
        X[rng.choice(60, 1 + j % 4, replace=False), j] = rng.standard_normal(1 + j % 4)
    return A, A @ X


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    from paper_1007_3753_b200.distributed import align_batch_sharded, solve_batch_sharded, src_classify_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, Bm = _problem()
        res = solve_batch_sharded(_oracle_batch, A, Bm, {"lam": 1e-3}, device="cpu")
        lab, cres = src_classify_sharded(_oracle_classify, A, None, Bm, None, device="cpu")
        Bs, bs = _align_problem()
        W, E = align_batch_sharded(_oracle_align, Bs, bs, {"tol": 1e-8}, device="cpu")
        np.savez(os.path.join(out_dir, "r%d.npz" % rank), x=res.x, it=res.iterations, conv=res.converged,
                 lam=res.lam, lab=lab, cres=cres, W=W, E=E)
    finally:
        dist.destroy_process_group()


def test_shard_indices_partition():
    from paper_1007_3753_b200.distributed import shard_indices
    for B in (1, 7, 64, 8192):
        for world in (1, 2, 3, 8):
            parts = [shard_indices(B, r, world) for r in range(world)]
            allj = np.sort(np.concatenate(parts))
            np.testing.assert_array_equal(allj, np.arange(B))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_batch_gathers_in_order(world):
    import torch.multiprocessing as mp
    A, Bm = _problem()
    full = _oracle_batch(A, Bm, {"lam": 1e-3})
    lab_ref, _, _ = _oracle_classify(A, None, Bm, None)
    W_ref, E_ref = _oracle_align(*_align_problem(), {"tol": 1e-8})
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), tmp), nprocs=world, join=True)
        outs = [dict(np.load(os.path.join(tmp, "r%d.npz" % r))) for r in range(world)]
    for o in outs:
        np.testing.assert_array_equal(o["x"], full.x)
        np.testing.assert_array_equal(o["it"], full.iterations)
        np.testing.assert_array_equal(o["conv"], full.converged)
        np.testing.assert_array_equal(o["lab"], lab_ref)
        np.testing.assert_array_equal(o["W"], W_ref)
        np.testing.assert_array_equal(o["E"], E_ref)
        # per-rank local indices were gathered back to their global slots
        from paper_1007_3753_b200.distributed import shard_indices
        for r in range(world):
            idx = shard_indices(Bm.shape[1], r, world)
            np.testing.assert_array_equal(o["lam"][idx], np.arange(idx.shape[0]) + 0.5)
            np.testing.assert_array_equal(o["cres"][idx, 0], np.arange(idx.shape[0]))


def _fail_worker(rank, world, port, out_dir):
    """Rank 1 fails inside its local solve: every rank must raise (ADVICE r01:
    no rank may be left blocked in the result gather)."""
    import torch.distributed as dist
    from paper_1007_3753_b200.distributed import solve_batch_sharded
    from paper_1007_3753_b200.exceptions import DeviceError, NumericalBreakdownError
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def solve(A, Bsub, config):
        if dist.get_rank() == 1:
            raise NumericalBreakdownError("rank 1 breaks down")
        return _oracle_batch(A, Bsub, config)
    try:
        A, Bm = _problem()
        try:
            solve_batch_sharded(solve, A, Bm[:, :3], {"lam": 1e-3}, device="cpu")
            outcome = "returned"
        except NumericalBreakdownError:
            outcome = "breakdown"
        except DeviceError:
            outcome = "peer_failed"
        with open(os.path.join(out_dir, "r%d.txt" % rank), "w") as fh:
            fh.write(outcome)
    finally:
        dist.destroy_process_group()


def test_sharded_batch_failure_raises_on_every_rank():
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_fail_worker, args=(3, _free_port(), tmp), nprocs=3, join=True)
        got = [open(os.path.join(tmp, "r%d.txt" % r)).read() for r in range(3)]
    assert got == ["peer_failed", "breakdown", "peer_failed"]


def test_batched_entry_points_accept_empty_share():
    """B < world leaves a rank with no columns: the batched entry points return
    an empty result instead of an argument error (no GPU needed for B = 0)."""
    from paper_1007_3753_b200 import batched
    from paper_1007_3753_b200.model import SolverConfig
    A = np.eye(4)
    r = batched._empty("fista", A, np.zeros((4, 0)), SolverConfig())
    assert r.x.shape == (4, 0) and r.results() == []
