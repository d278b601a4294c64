"""The config-4 dictionary passes alone, for ncu: one 8-way shard of the
config-4 instance (d=65536, 32768 columns, fp32, 8 GiB — the per-GPU share
at 8 GPUs; >> L2 like the full 64 GiB) and a few launches of each pass.

    ncu --set full -k regex:"gemv_partial|gemv_t_stream" -c 4 python tools/cfg4_kernels.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1007_3753_b200.sharded import make_cfg4_shard  # noqa: E402

class _Solo:
    """rank 0 of an S-way split, no peers (the collective is not profiled)."""
    world = int(os.environ.get("SHARDS", "8"))
    rank = 0
    group = None

    def allreduce_(self, t):
        pass

    def all_gather(self, t):
        return t.repeat(self.world)


shard, b, x0, ops = make_cfg4_shard(rank=0, world=_Solo.world, coll=_Solo())
x = ops.zeros_n()
x.normal_()
r = ops.from_host_d(b)
y = ops.zeros_d()
g = ops.zeros_n()
for _ in range(int(os.environ.get("REPS", "2"))):
    ops.gemv(x, y)
    ops.gemv_t(r, g)
torch.cuda.synchronize()
print("shard bytes", shard.local.n * shard.d * 4)
