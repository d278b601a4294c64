"""Batches sharded across GPUs (configs 3 and 5).

Instances are independent, so the batch is split across the ranks of a
torch.distributed group (one process per GPU, A — and the dual solver's Gram
factor — replicated on every GPU) and each rank runs the batched solver on
its share with no per-iteration communication.  One all-gather at the end
assembles x / iterations / converged / status (and, for Homotopy, the lambda
reached; for SRC, the labels) in the original instance order on every rank.

Instances are dealt round-robin (instance j -> rank j mod world) so ranks
get the same mix of sparsity levels — per-instance iteration counts vary
with k, and contiguous blocks would leave the ranks with the sparse
instances idle at the end.
"""

import numpy as np


def _world(group):
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(group), dist.get_rank(group)
    except ImportError:
        pass
    return 1, 0


def shard_indices(B, rank, world):
    """Instances owned by `rank` (round-robin deal, ascending)."""
    return np.arange(rank, int(B), int(world), dtype=np.int64)


def _gather_rows(arr, B, world, group, device):
    """All-gather per-rank row blocks (rank r holds rows r, r+world, ...) into
    the full (B, ...) array on every rank."""
    import torch
    import torch.distributed as dist
    arr = np.ascontiguousarray(arr)
    cap = (B + world - 1) // world
    tail = arr.shape[1:]
    buf = np.zeros((cap,) + tail, dtype=arr.dtype)
    buf[: arr.shape[0]] = arr
    t = torch.from_numpy(buf).to(device)
    outs = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    full = np.zeros((B,) + tail, dtype=arr.dtype)
    for r in range(world):
        idx = shard_indices(B, r, world)
        full[idx] = outs[r].cpu().numpy()[: idx.shape[0]]
    return full


def _collective_call(fn, world, group, device):
    """Run the rank-local ``fn()``; before any result collective, all ranks
    agree (MAX all-reduce of a failure flag) on whether some rank failed, so a
    failure on one rank raises on every rank instead of leaving the others
    blocked in the gather."""
    if world == 1:
        return fn()
    import torch
    import torch.distributed as dist
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
    out, err = None, None
    try:
        out = fn()
    except Exception as exc:  # noqa: BLE001 - re-raised after the agreement below
        err = exc
    flag = torch.tensor([1 if err is not None else 0], dtype=torch.int32, device=device)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if err is not None:
        raise err
    if int(flag.item()):
        from paper_1007_3753_b200.exceptions import DeviceError
        raise DeviceError("the batched solve failed on another rank")
    return out


def solve_batch_sharded(solve, A, Bmat, config, group=None, device=None, **kw):
    """Run ``solve(A, Bmat_share, config, **kw)`` (a batched entry point such as
    batched.fista_solve_batch / dalm_solve_batch / homotopy_solve_batch) on
    this rank's share of the columns of Bmat (d x B) and return the full
    BatchResult (original order) on every rank.  ``device``: where the
    collective buffers live (the rank's CUDA device under NCCL, "cpu" under
    gloo)."""
    from paper_1007_3753_b200.batched import BatchResult
    Bmat = np.asarray(Bmat, dtype=np.float64)
    B = Bmat.shape[1]
    world, rank = _world(group)
    idx = shard_indices(B, rank, world)
    res = _collective_call(lambda: solve(A, np.ascontiguousarray(Bmat[:, idx]), config, **kw),
                           world, group, device)
    if world == 1:
        return res
    if device is None:
        import torch
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
    x = _gather_rows(res.x.T, B, world, group, device).T
    its = _gather_rows(np.asarray(res.iterations, np.int64), B, world, group, device)
    conv = _gather_rows(np.asarray(res.converged, np.int64), B, world, group, device)
    stat = _gather_rows(np.asarray(res.status, np.int64), B, world, group, device)
    trace = None
    if res.trace is not None:
        trace = _gather_rows(res.trace, B, world, group, device)
    out = BatchResult(np.ascontiguousarray(x), its.astype(np.int32), conv.astype(np.int32),
                      stat.astype(np.int32), res.wall_time_seconds, trace, res.kind, res.max_iter)
    if getattr(res, "lam", None) is not None:
        out.lam = _gather_rows(np.asarray(res.lam, np.float64), B, world, group, device)
    if getattr(res, "notes", None) is not None:
        out.notes = _gather_rows(np.asarray(res.notes, np.int64), B, world, group, device).astype(np.int32)
    return out


def src_classify_sharded(classify, A, class_labels, Bmat, config, group=None, device=None):
    """SRC over a query batch split across ranks: ``classify`` is
    batched.src_classify; returns (labels, class_residuals) for all queries on
    every rank."""
    Bmat = np.asarray(Bmat, dtype=np.float64)
    B = Bmat.shape[1]
    world, rank = _world(group)
    idx = shard_indices(B, rank, world)
    labels, resid, _ = _collective_call(
        lambda: classify(A, class_labels, np.ascontiguousarray(Bmat[:, idx]), config), world, group, device)
    if world == 1:
        return np.asarray(labels), np.asarray(resid)
    if device is None:
        import torch
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
    lab = _gather_rows(np.asarray(labels, np.int64), B, world, group, device)
    res = _gather_rows(np.asarray(resid, np.float64), B, world, group, device)
    return lab.astype(np.int32), res


def align_batch_sharded(solve, Bs, bs, config, group=None, device=None, **kw):
    """Alignment images split across ranks (SURVEY §8(f) rank 4 on §8(e)'s
    batch sharding): ``solve`` is robust.align_*_solve_batch, Bs (count, d, m),
    bs (count, d); every rank gets (W, E) for all images in the original order."""
    Bs = np.asarray(Bs, dtype=np.float64)
    bs = np.asarray(bs, dtype=np.float64)
    count = Bs.shape[0]
    world, rank = _world(group)
    idx = shard_indices(count, rank, world)
    W, E = _collective_call(lambda: solve(np.ascontiguousarray(Bs[idx]), np.ascontiguousarray(bs[idx]),
                                          config, **kw), world, group, device)
    if world == 1:
        return W, E
    if device is None:
        import torch
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
    return (_gather_rows(np.asarray(W), count, world, group, device),
            _gather_rows(np.asarray(E), count, world, group, device))
