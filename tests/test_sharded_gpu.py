"""Column-sharded FISTA on the GPU (world size 1 on this box; the N>1 control
flow is covered by tests/test_sharded_cpu.py over gloo) plus the shard
primitives ell1_gemv / ell1_gemv_t against numpy, including the long-column
GEMV^T path (ld / vector width > 512)."""

import ctypes

import numpy as np
import pytest

from tests.gpu_util import assert_parity, case_inputs, make_config

pytestmark = pytest.mark.gpu


def _dev_dict(A, dtype):
    from paper_1007_3753_b200 import device
    return device.DeviceDictionary(A, dtype=dtype)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("shape", [(20, 40), (500, 1000), (1024, 4096), (1500, 700),
                                   (4100, 300), (9000, 2000), (65536, 64)])
def test_gemv_pair(shape, dtype):
    import torch
    from paper_1007_3753_b200 import _lib, device
    d, n = shape
    rng = np.random.default_rng(d * 7 + n)
    A = rng.standard_normal((d, n))
    D = _dev_dict(A, dtype)
    Ah = A if dtype == "float64" else A.astype(np.float32).astype(np.float64)
    L = _lib.lib()
    v = D.view()
    wsb = L.ell1_gemv_workspace(ctypes.byref(v))
    ws = device.alloc_bytes(wsb, D.device)
    x = rng.standard_normal(n)
    r = rng.standard_normal(d)
    xd = device.to_device_vec(x, n, D.device)
    rd = device.to_device_vec(r, D.ld, D.device)
    y = torch.zeros(D.ld, dtype=torch.float64, device=D.device)
    g = torch.zeros(n, dtype=torch.float64, device=D.device)
    st = device.stream_ptr(D.device)
    _lib.check(L.ell1_gemv(ctypes.byref(v), device.ptr(xd), device.ptr(y), device.ptr(ws), wsb, st),
               "gemv")
    _lib.check(L.ell1_gemv_t(ctypes.byref(v), device.ptr(rd), device.ptr(g), device.ptr(ws), wsb,
                             st), "gemv_t")
    yh = y.cpu().numpy()[:d]
    gh = g.cpu().numpy()
    tol = 1e-12
    np.testing.assert_allclose(yh, Ah @ x, rtol=0, atol=tol * np.abs(Ah).sum(1).max() * 4)
    np.testing.assert_allclose(gh, Ah.T @ r, rtol=0, atol=tol * np.abs(Ah).sum(0).max() * 4)


CASES = ["fista_small_1400", "fista_small_exactL", "fista_small_relobj", "fista_small_gtrule",
         "fista_small_noncont", "fista_qr", "cfg1_fista", "cfg2_fista"]


@pytest.mark.parametrize("cid", CASES)
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_sharded_fista_device_world1(cid, dtype):
    from paper_1007_3753_b200.sharded import ShardedDictionary, ShardedInstance, sharded_fista_solve
    case, A, b, gt, gold = case_inputs(cid)
    cfg = make_config(case, A, b, dtype=dtype)
    shard = ShardedDictionary.from_dense(A, 0, 1, dtype=dtype)
    res = sharded_fista_solve(ShardedInstance(shard, b, gt), cfg)
    if dtype == "float64":
        assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-6)
    else:
        from tests.gpu_util import rel_err, support
        assert rel_err(res.x_star, gold["x"]) <= 1e-4
        assert support(res.x_star) == support(gold["x"])
        assert bool(res.converged) == bool(gold["converged"])


def test_sharded_matches_single_gpu_fista():
    """The sharded driver and the persistent single-instance kernel agree."""
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    from paper_1007_3753_b200.sharded import ShardedDictionary, ShardedInstance, sharded_fista_solve
    from paper_1007_3753_b200.shrinkage import fista_solve
    from paper_1007_3753_b200.synth import make_problem, Workload
    P = make_problem(Workload("long", 3000, 8000, 150, seed=11, noise_rel=0.01))
    cfg = SolverConfig(lam=None, tol=1e-6, max_iter=3000,
                       stopping=StoppingRule("relative-estimate", 1e-6))
    a = fista_solve(P, cfg)
    shard = ShardedDictionary.from_dense(P.A, 0, 1)
    b = sharded_fista_solve(ShardedInstance(shard, P.b), cfg)
    assert abs(a.iterations - b.iterations) <= 1
    den = np.linalg.norm(a.x_star)
    assert np.linalg.norm(a.x_star - b.x_star) <= 1e-6 * den
