"""Host (numpy + gloo) implementation of the ShardOps interface of
paper_1007_3753_b200/sharded.py — TEST INFRASTRUCTURE ONLY.

It lets the CPU suite drive the column-sharded FISTA control loop at
world_size 1..3 over torch.distributed/gloo and compare it with the oracle
and the reference's golden outputs.  The product path (DeviceShardOps) never
touches this module; the elementwise formulas restate csrc/shard.cu.
"""

import numpy as np

from oracle.l1_oracle import soft


class NumpyShardOps:
    def __init__(self, A_local, group=None):
        import torch.distributed as dist
        self.A = np.ascontiguousarray(A_local, dtype=np.float64)
        self.d, self.nl = self.A.shape
        self.ld = self.d
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        self.mine = np.zeros(8)
        self.rsum = np.zeros(8)

    def zeros_d(self):
        return np.zeros(self.d)

    def zeros_n(self):
        return np.zeros(self.nl)

    def from_host_d(self, v):
        return np.array(v, dtype=np.float64)

    def from_host_n(self, v):
        return np.array(v, dtype=np.float64)

    def to_host_n(self, v):
        return v.copy()

    def to_host_d(self, v):
        return v.copy()

    def gemv(self, x, out):
        out[:] = self.A @ x

    def gemv_t(self, r, out):
        out[:] = self.A.T @ r

    def prox(self, x, xp, gx, gxp, xn, m, L, lam, gt):
        y = x + m * (x - xp)
        g = (1.0 + m) * gx - m * gxp
        u = soft(y - g / L, lam / L)
        dl = u - y
        s = np.zeros(8)
        s[0] = np.sum(np.abs(u))
        s[1] = g @ dl
        s[2] = dl @ dl
        s[3] = np.max(np.abs(u)) if u.size else 0.0
        s[4] = (u - x) @ (u - x)
        s[5] = x @ x
        if gt is not None:
            s[6] = (u - gt) @ (u - gt)
        xn[:] = u
        self.mine = s

    def resid(self, ax, b, rx, mn, rn):
        r = ax - b
        ry = (1.0 + mn) * r - mn * rx
        self.rsum = np.array([r @ r, ry @ ry, 0, 0, 0, 0, 0, 0], dtype=np.float64)
        rn[:] = r

    def kkt(self, x, g, lam, cut):
        c = -g
        on = x != 0.0
        s = np.zeros(8)
        if np.any(on):
            s[0] = np.max(np.abs(c[on] - lam * np.sign(x[on])))
            s[2] = 1.0
        if np.any(~on):
            s[1] = np.max(np.abs(c[~on]))
            s[3] = 1.0
        s[4] = float(np.count_nonzero(np.abs(x) > cut))
        self.mine = s

    def allreduce_(self, v):
        if self.world > 1:
            import torch
            import torch.distributed as dist
            t = torch.from_numpy(v)
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def _gather(self):
        if self.world == 1:
            return self.mine.reshape(1, 8).copy()
        import torch
        import torch.distributed as dist
        outs = [torch.zeros(8, dtype=torch.float64) for _ in range(self.world)]
        dist.all_gather(outs, torch.from_numpy(self.mine.copy()), group=self.group)
        return np.stack([o.numpy() for o in outs])

    def trial_scalars(self):
        return self._gather(), self.rsum.copy()

    def kkt_scalars(self):
        return self._gather()

    def gather_n(self, v, n_global):
        if self.world == 1:
            return v.copy()
        import torch
        import torch.distributed as dist
        from paper_1007_3753_b200.sharded import column_range
        sizes = [column_range(n_global, r, self.world) for r in range(self.world)]
        cap = max(c1 - c0 for c0, c1 in sizes)
        buf = torch.zeros(cap, dtype=torch.float64)
        buf[: self.nl] = torch.from_numpy(v)
        outs = [torch.zeros(cap, dtype=torch.float64) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        return np.concatenate([outs[r].numpy()[: c1 - c0] for r, (c0, c1) in enumerate(sizes)])
