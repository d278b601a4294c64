"""Several "ranks" of the column-sharded FISTA on ONE GPU — TEST
INFRASTRUCTURE ONLY.

Each rank is a host thread with its own DeviceShardOps (its own column
panel, vectors and device control block); the collective is a host barrier:
every rank synchronises the device, rank 0 sums the deposited tensors in
rank order, every rank copies the sum back.  No kernel ever waits on another
rank's kernel (the only cross-rank dependency is this host-side exchange),
so this exercises the product's multi-rank device code — slot packing, the
rank-order folds, identical decisions on every rank, result assembly — with
world > 1 on the single GPU this environment has.
"""

import threading


class SharedGroup:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.bufs = [None] * world
        self.out = None
        self.calls = 0

    def _sync(self):
        import torch
        torch.cuda.synchronize()

    def allreduce(self, rank, t):
        self._sync()
        self.bufs[rank] = t
        self.barrier.wait()
        if rank == 0:
            s = self.bufs[0].clone()
            for r in range(1, self.world):
                s += self.bufs[r]
            self._sync()
            self.out = s
            self.calls += 1
        self.barrier.wait()
        t.copy_(self.out)
        self._sync()
        self.barrier.wait()

    def all_gather(self, rank, t):
        import torch
        self._sync()
        self.bufs[rank] = t
        self.barrier.wait()
        if rank == 0:
            self.out = torch.cat([b.clone() for b in self.bufs])
            self._sync()
        self.barrier.wait()
        out = self.out.clone()
        self._sync()
        self.barrier.wait()
        return out


class ThreadCollective:
    def __init__(self, shared, rank):
        self.shared = shared
        self.world = shared.world
        self.rank = rank
        self.group = None

    def allreduce_(self, t):
        self.shared.allreduce(self.rank, t)

    def all_gather(self, t):
        return self.shared.all_gather(self.rank, t)


def run_ranks(world, fn):
    """fn(rank, coll) on `world` threads; returns the per-rank results
    (re-raises the first exception)."""
    shared = SharedGroup(world)
    out = [None] * world
    err = [None] * world

    def body(r):
        try:
            out[r] = fn(r, ThreadCollective(shared, r))
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            err[r] = exc
            shared.barrier.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return out, shared
