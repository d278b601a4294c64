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
                                   (4100, 300), (9000, 2000), (65536, 64), (8192, 3001), (40960, 37),
                                   (131072, 21)])
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


# ---------------------------------------------------------------- world > 1 on one GPU
def _emulated_solve(A, b, cfg, world, dtype="float64", gt=None):
    """The product's DeviceShardOps on `world` thread-ranks of this GPU
    (tests/emulated_collective.py): every rank returns its SolverResult."""
    from paper_1007_3753_b200.sharded import (DeviceShardOps, ShardedDictionary, ShardedInstance,
                                              sharded_fista_solve)
    from tests.emulated_collective import run_ranks

    def rank_fn(rank, coll):
        import torch
        torch.cuda.set_device(0)
        shard = ShardedDictionary.from_dense(A, rank, world, dtype=dtype)
        ops = DeviceShardOps(shard, coll)
        return sharded_fista_solve(ShardedInstance(shard, b, gt), cfg, ops=ops)
    return run_ranks(world, rank_fn)


@pytest.mark.parametrize("cid", ["fista_small_1400", "fista_small_relobj", "fista_small_kktrule",
                                 "fista_small_gtrule", "fista_small_budget", "fista_small_noncont",
                                 "cfg1_fista", "cfg2_fista"])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fista_emulated_ranks_match_golden(cid, world):
    """world > 1: slot packing, rank-order folds and identical device
    decisions on every rank; each rank returns the reference's result."""
    case, A, b, gt, gold = case_inputs(cid)
    cfg = make_config(case, A, b)
    results, shared = _emulated_solve(A, b, cfg, world, gt=gt)
    for res in results:
        assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-6)
    for res in results[1:]:
        np.testing.assert_array_equal(res.x_star, results[0].x_star)


def test_sharded_fista_one_collective_per_round():
    """The data path exchanges exactly one allreduce per round (plus the
    set-up slot exchange and the final x all-gather)."""
    from paper_1007_3753_b200.sharded import (DeviceShardOps, ShardedDictionary, ShardedFista)
    from tests.emulated_collective import run_ranks
    case, A, b, gt, gold = case_inputs("cfg1_fista")
    cfg = make_config(case, A, b)
    rounds = []

    def rank_fn(rank, coll):
        shard = ShardedDictionary.from_dense(A, rank, 2)
        drv = ShardedFista(DeviceShardOps(shard, coll), b, A.shape[1], cfg)
        res = drv.solve()
        rounds.append(drv.rounds)
        return res
    results, shared = run_ranks(2, rank_fn)
    assert rounds[0] == rounds[1]
    assert shared.calls == rounds[0] + 1            # rounds + the set-up slot exchange
    assert results[0].iterations == int(gold["iterations"])


def test_sharded_rejects_foreign_column_split():
    from paper_1007_3753_b200 import device
    from paper_1007_3753_b200.sharded import DeviceShardOps, ShardedDictionary
    A = np.random.default_rng(0).standard_normal((20, 40))
    D = device.DeviceDictionary(A[:, 3:30])
    with pytest.raises(ValueError):
        DeviceShardOps(ShardedDictionary(D, 3, 40))


# ---------------------------------------------------------------- config-4 proxy vs the reference
def _cfg4_proxy():
    import json
    import os
    from paper_1007_3753_b200 import synth
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg4_proxy_fista.npz"))
    rc = json.loads(str(g["recipe"]))
    A = synth.gen_gaussian_dict(rc["d"], rc["n"], rc["seed"])
    return A, g["b"], g


@pytest.mark.parametrize("world,dtype", [(1, "float64"), (2, "float64"), (4, "float64"),
                                         (1, "float32"), (2, "float32")])
def test_cfg4_proxy_matches_reference(world, dtype):
    """Scaled config-4 proxy (d=8192, n=32768, k=256, 1e-3 relative noise,
    default lambda, relative-estimate 1e-6) through the sharded path against
    the real reference fista_solve (tests/golden/make_scale_golden.py):
    fp64 bit-for-bit control flow (same iterations and trace), x within
    1e-6; fp32 storage within 1e-4 and the same support; 1-vs-N agreement."""
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    from tests.gpu_util import rel_err, support
    A, b, gold = _cfg4_proxy()
    cfg = SolverConfig(lam=None, tol=1e-6, max_iter=5000,
                       stopping=StoppingRule("relative-estimate", 1e-6), options={"dtype": dtype})
    results, _ = _emulated_solve(A, b, cfg, world, dtype=dtype)
    res = results[0]
    if dtype == "float64":
        assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-6)
    else:
        assert rel_err(res.x_star, gold["x"]) <= 1e-4
        assert support(res.x_star) == support(gold["x"])
        assert abs(res.iterations - int(gold["iterations"])) <= 2
    for r in results[1:]:
        np.testing.assert_array_equal(r.x_star, res.x_star)


def test_cfg4_full_scale_kkt_certificate():
    """BASELINE config 4 at full size (d=65536, n=262144, fp32 storage,
    64 GiB) on one GPU: the solve converges under the headline rule and an
    independent fp64 recomputation of c = A^T (b - A x) certifies the
    solution (model.kkt_from_correlation <= 1e-3 lambda, model.py:160-173);
    the objective matches the last trace row, the large entries of x0 are
    all recovered."""
    import torch
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    from paper_1007_3753_b200.sharded import (ShardedInstance, kkt_certificate, make_cfg4_shard,
                                              sharded_fista_solve)
    free, _ = torch.cuda.mem_get_info()
    if free < 72 * 2 ** 30:
        pytest.skip("needs ~70 GiB of free device memory")
    shard, b, x0, ops = make_cfg4_shard()
    cfg = SolverConfig(lam=None, tol=1e-6, max_iter=2000, stopping=StoppingRule("relative-estimate", 1e-6))
    res = sharded_fista_solve(ShardedInstance(shard, b), cfg, ops=ops)
    assert res.converged and 10 < res.iterations < 2000
    lam = 1e-2 * ops.setup(b)            # default lambda = 1e-2 ||A^T b||_inf
    kk, F = kkt_certificate(ops, res.x_star, b, lam)
    assert kk <= 1e-3 * lam, (kk, lam)
    assert abs(F - res.trace[-1].objective) <= 1e-9 * abs(F)
    big = np.abs(x0) > 4 * lam
    assert np.all(res.x_star[big] != 0.0)
    del ops, shard
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- column-sharded Homotopy (§8(e) row 3)
@pytest.mark.parametrize("cid", ["homotopy_small_1300", "homotopy_small_1301", "cfg2_homotopy",
                                 "cfg5_homotopy_k16", "cfg5_homotopy_k64"])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_homotopy_matches_golden(cid, world):
    """The sharded path (A^T passes per rank, replicated active set and
    factor on the device) on `world` thread-ranks of this GPU against the
    reference's golden path: same breakpoints, trace and x (fp64)."""
    from tests.golden.cases import resolve_lambda
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.sharded import ShardedDictionary, ShardedInstance
    from paper_1007_3753_b200.sharded_homotopy import DeviceHomShardOps, sharded_solve_path
    from tests.emulated_collective import run_ranks
    case, A, b, gt, gold = case_inputs(cid)
    lam = resolve_lambda(case["cfg"], A, b)
    target = lam if lam is not None else 1e-2 * float(np.max(np.abs(A.T @ b)))

    def rank_fn(rank, coll):
        import torch
        torch.cuda.set_device(0)
        shard = ShardedDictionary.from_dense(A, rank, world)
        return sharded_solve_path(ShardedInstance(shard, b), target, SolverConfig(max_iter=5000),
                                  ops=DeviceHomShardOps(shard, coll))
    results, _ = run_ranks(world, rank_fn)
    for res, lam_r in results:
        assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-8)
        np.testing.assert_array_equal(res.x_star, results[0][0].x_star)


def test_gemv_stream_pass_at_16gib():
    """The streamed A x pass that config 4's >= 16 GiB dictionaries take
    (shard.cu gemv_stream_kernel + the fixed-order row reduction) and the
    grouped streamed A^T r pass, against a chunked fp64 torch product on a
    65536 x 65536 fp32 dictionary (16 GiB), and A x against the engine panel
    pass (ELL1_GEMV_PANEL) to rounding level."""
    import os
    import torch
    from paper_1007_3753_b200 import _lib, device
    dev = torch.device("cuda", 0)
    d = n = 65536
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    st = torch.empty(n, d, device=dev, dtype=torch.float32)
    for c0 in range(0, n, 8192):
        st[c0:c0 + 8192].normal_(generator=g)
    D = device.DeviceDictionary.wrap(st, d)
    v = D.view()
    L = _lib.lib()
    wsb = L.ell1_gemv_workspace(ctypes.byref(v))
    ws = device.alloc_bytes(wsb, dev)
    x = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
    r = torch.randn(D.ld, dtype=torch.float64, device=dev, generator=g)
    y = torch.zeros(D.ld, dtype=torch.float64, device=dev)
    y2 = torch.zeros(D.ld, dtype=torch.float64, device=dev)
    gg = torch.zeros(n, dtype=torch.float64, device=dev)
    s = device.stream_ptr(dev)
    _lib.check(L.ell1_gemv(ctypes.byref(v), device.ptr(x), device.ptr(y), device.ptr(ws), wsb, s), "gemv")
    _lib.check(L.ell1_gemv_t(ctypes.byref(v), device.ptr(r), device.ptr(gg), device.ptr(ws), wsb, s), "gemv_t")
    os.environ["ELL1_GEMV_PANEL"] = "1"
    try:
        _lib.check(L.ell1_gemv(ctypes.byref(v), device.ptr(x), device.ptr(y2), device.ptr(ws), wsb, s), "gemv")
    finally:
        del os.environ["ELL1_GEMV_PANEL"]
    yref = torch.zeros(d, dtype=torch.float64, device=dev)
    gref = torch.empty(n, dtype=torch.float64, device=dev)
    for c0 in range(0, n, 4096):
        blk = st[c0:c0 + 4096].double()                       # (4096 columns) x d, row-major = A[:, c].T
        yref += blk.t() @ x[c0:c0 + 4096]
        gref[c0:c0 + 4096] = blk @ r[:d]
        del blk
    torch.cuda.synchronize()
    scale_y = float(torch.abs(st).sum(0).max()) * float(torch.abs(x).max())
    scale_g = float(torch.abs(st).sum(1).max()) * float(torch.abs(r).max())
    assert float(torch.abs(y[:d] - yref).max()) <= 1e-13 * scale_y
    assert float(torch.abs(y[:d] - y2[:d]).max()) <= 1e-13 * scale_y
    assert float(torch.abs(gg - gref).max()) <= 1e-13 * scale_g


def test_fista_solve_streams_large_fp32_dictionaries():
    """shrinkage.fista_solve on a >= 1 GiB float32 dictionary (the config-4
    proxy, d=8192, n=32768) takes the streaming route (the sharded rounds at
    world 1): same answer as the persistent kernel and as the reference
    golden; an observer keeps the persistent kernel."""
    from paper_1007_3753_b200 import shrinkage
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig, StoppingRule
    from tests.gpu_util import rel_err, support
    A, b, gold = _cfg4_proxy()
    cfg = SolverConfig(lam=None, tol=1e-6, max_iter=5000,
                       stopping=StoppingRule("relative-estimate", 1e-6), options={"dtype": "float32"})
    P = ProblemInstance(A, b)
    assert shrinkage._stream_route(P, cfg, None)
    assert not shrinkage._stream_route(P, cfg, lambda *a: None)
    routed = shrinkage.fista_solve(P, cfg)
    engine = shrinkage.FistaPlan(P, cfg).solve(None)
    assert routed.iterations == engine.iterations
    assert rel_err(routed.x_star, engine.x_star) <= 1e-9
    assert [t.iteration for t in routed.trace] == [t.iteration for t in engine.trace]
    assert rel_err(routed.x_star, gold["x"]) <= 1e-4
    assert support(routed.x_star) == support(gold["x"])
