#!/usr/bin/env python
"""Benchmark: BASELINE config 4 — one d=65536 x n=262144 compressed-sensing
instance (fp32 storage, 64 GiB), FISTA with default lambda and relative
change in x < 1e-6, column-sharded over the ranks with ONE allreduce per
backtracking trial and all control on the device.  One step = one complete
solve; the metric is solver iterations/s of the whole job (config 4 is one
instance: total work fixed, strong scaling).

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]

--gpus N without torchrun re-launches itself under torch.distributed.run
(one rank per GPU, NCCL).  --impl reference times the reference algorithm's
CPU implementation (the numpy/OpenBLAS port of shrinkage.fista_solve, all
host cores) on a scaled proxy of the same instance (d=8192, n=32768, fp64 —
the reference is fp64-only and a 64 GiB dictionary does not fit its host
path) and extrapolates by dictionary bytes (x64).  --dry-run drives the
launcher, the gloo rendezvous and the sharded control protocol on CPU
(numpy shard ops, small proxy) — no GPU, no timing claim.

Secondary legs (N=1): configs 1, 2 (all solvers), 3, 5, the HBM streaming
roofline, the experiment harness and the alignment solvers.
"""

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "l1-min solver iterations/sec (config 4: one 65536 x 262144 instance, FISTA)"
UNIT = "iterations/s"
WORKLOAD = ("cfg4: single compressed-sensing instance d=65536 n=262144 (A fp32 storage, 64 GiB, unit-norm "
            "Gaussian columns), k=2048 N(0,1), b = A x0 + 1e-3 relative noise; FISTA, lambda = "
            "1e-2||A^T b||_inf, stop relative-estimate 1e-6 (max_iter 2000); column-sharded, one NCCL "
            "allreduce of [A_r x_r | scalar slots] per backtracking trial")
PROXY = dict(d=8192, n=32768, k=256, seed=4, noise_rel=1e-3)      # = tests/golden cfg4_proxy_fista
PROXY_SCALE = (65536 * 262144) / (8192 * 32768)                  # dictionary-bytes ratio (64)
CFG2_WORKLOAD = ("cfg2: single noisy BPDN instance d=1024 n=4096 k=128 sigma=0.01||Ax0||/sqrt(d), "
                 "FISTA, lambda=1e-2||A^T b||_inf, stop relative-estimate 1e-6")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo dry run of the launcher + protocol")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-stream", action="store_true", help="skip the HBM streaming roofline leg")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the config 1/2/3/5 and all-solver legs")
    ap.add_argument("--cfg5-sweep", action="store_true", help="add the config-5 batch-size sweep leg")
    ap.add_argument("--only-leg", default=None, help="run one secondary leg alone (diagnostics)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_launch(args):
    """--gpus N > 1 outside torchrun: re-run this script under
    torch.distributed.run with N ranks on this node (rendezvous on
    127.0.0.1); NCCL's init lines (rings, NVLS) go to stderr."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    env = dict(os.environ)
    if not args.dry_run and "NCCL_DEBUG" not in env:
        env.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT,NVLS", NCCL_DEBUG_FILE="/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node=%d" % args.gpus, "--master-addr=127.0.0.1",
           "--master-port=%d" % _free_port(), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def make_instance(rank):
    from paper_1007_3753_b200 import synth
    w = synth.Workload("cfg2", 1024, 4096, 128, seed=rank, noise_rel=0.01)
    return synth.make_problem(w)


def config(dtype="float64"):
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    return SolverConfig(lam=None, tol=1e-6, stopping=StoppingRule("relative-estimate", 1e-6),
                        options={"dtype": dtype})


def cfg4_config(max_iter=2000):
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    return SolverConfig(lam=None, tol=1e-6, max_iter=max_iter,
                        stopping=StoppingRule("relative-estimate", 1e-6))


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_ready(self, timeout=10.0):
        """Block until nvidia-smi has produced its first sample."""
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        loaded = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- CPU legs
def cpu_solve_once(P):
    import oracle  # CPU baseline / reference arm only
    return oracle.fista(P.A, P.b, lam=None, tol=1e-6, stop=("relative-estimate", 1e-6))


def _pool_init():
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)                       # one BLAS thread per worker process


def _cpu_task(args):
    """One reference-port solve in a worker (SURVEY §8(d) batched CPU baseline)."""
    import oracle  # CPU baseline only
    kind, A, b = args[:3]
    if kind == "fista":
        return oracle.fista(A, b, lam=1e-3, tol=1e-6, stop=("relative-estimate", 1e-6)).iterations
    if kind == "dalm":
        return oracle.dalm(A, b, tol=1e-6, stop=("relative-estimate", 1e-6)).iterations
    if kind == "homotopy":
        return oracle.homotopy(A, b, 1e-3)[0].iterations
    if kind == "cab_dalm":
        return oracle.cab(A, b, "dalm", tol=1e-4, max_iter=2000)[2].iterations
    if kind == "align_palm":                              # A = B (d x m), b = the image
        from oracle.l1_oracle import align_palm
        align_palm(A, b, tol=1e-8, max_iter=5000)
        return 1
    if kind.startswith("harness_"):                       # one phase-grid trial, lambda = args[3]
        lam = args[3]
        if kind == "harness_fista":
            return oracle.fista(A, b, lam=lam, tol=1e-8, max_iter=20000).iterations
        if kind == "harness_homotopy":
            return oracle.homotopy(A, b, lam, max_iter=20000)[0].iterations
        return oracle.dalm(A, b, tol=1e-8, max_iter=20000).iterations
    raise ValueError(kind)


def _pool_warm(_):
    import oracle  # noqa: F401  (CPU baseline only: imports paid before the timed map)
    time.sleep(0.05)                           # keeps the warm-up spread over every worker
    return os.getpid()


def cpu_pool_tasks(tasks):
    """(instances/s, iterations/s, seconds, cores) of the oracle port over a
    process pool of all host cores, one BLAS thread per worker.  The pool is
    started and every worker has imported the port before the clock starts,
    and the tasks go out one at a time (chunksize 1, the reference harness's
    pattern), so the rate is solve time, not process start-up."""
    from concurrent.futures import ProcessPoolExecutor
    cores = os.cpu_count()
    with ProcessPoolExecutor(max_workers=cores, initializer=_pool_init) as ex:
        list(ex.map(_pool_warm, range(4 * cores)))
        t0 = time.perf_counter()
        its = list(ex.map(_cpu_task, tasks))
        el = time.perf_counter() - t0
    return len(tasks) / el, float(sum(its)) / el, el, cores


def cpu_pool_rate(kind, A, cols, per_core=4):
    """Instances/s of the reference port over a process pool of all host cores
    (one BLAS thread each, the reference bench's _run_tasks pattern) on
    per_core x cores instances of the batch."""
    count = min(per_core * os.cpu_count(), len(cols))
    rate, irate, el, cores = cpu_pool_tasks([(kind, A, cols[j]) for j in range(count)])
    return {"solves_per_sec": rate, "iterations_per_sec": irate, "instances": count,
            "seconds": el, "cores": cores, "kind": "port",
            "sample": "first %d instances of the batch, ProcessPoolExecutor(%d warm workers, 1 BLAS thread each)"
                      % (count, cores)}


def cpu_baseline_cfg2(P, budget_s=10.0):
    n = 0
    t0 = time.perf_counter()
    its = 0
    while True:
        r = cpu_solve_once(P)
        its += r.iterations
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s and n >= 2:
            break
    return {"value": n / el, "unit": "solves/s", "cores": os.cpu_count(), "kind": "port",
            "sample": "%d full cfg2 FISTA solves (numpy/OpenBLAS oracle port of "
                      "shrinkage.fista_solve, %d iterations total) in %.1f s" % (n, its, el),
            "iterations_per_sec": its / el}


def proxy_problem():
    from paper_1007_3753_b200 import synth
    w = synth.Workload("cfg4p", PROXY["d"], PROXY["n"], PROXY["k"], PROXY["seed"], PROXY["noise_rel"])
    return synth.make_problem(w)


def cpu_cfg4_sample(P, iters):
    """`iters` FISTA iterations of the oracle port (shrinkage.fista_solve
    restated, numpy/OpenBLAS on all host cores) on the config-4 proxy;
    returns (seconds, iterations, passes-equivalent)."""
    import oracle  # CPU baseline / reference arm only
    t0 = time.perf_counter()
    r = oracle.fista(P.A, P.b, lam=None, tol=1e-6, max_iter=iters, stop=("relative-estimate", 1e-6))
    return time.perf_counter() - t0, int(r.iterations)


def cpu_baseline_cfg4(budget_s=15.0):
    P = proxy_problem()
    cpu_cfg4_sample(P, 2)                      # warm (BLAS threads, page-in)
    t, its, n = 0.0, 0, 0
    while t < budget_s or n < 1:
        dt, k = cpu_cfg4_sample(P, 8)
        t += dt
        its += k
        n += 1
    v = its / t / PROXY_SCALE
    return {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": "%d x 8 FISTA iterations (oracle port of shrinkage.fista_solve, numpy/OpenBLAS, "
                      "fp64) on the d=8192 n=32768 proxy of config 4 in %.1f s; iterations/s divided by "
                      "the dictionary-bytes ratio %d (streaming-bound on the host)" % (n, t, PROXY_SCALE),
            "proxy_iterations_per_sec": its / t}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    P = proxy_problem()
    per_step = 4
    for _ in range(args.warmup):
        cpu_cfg4_sample(P, per_step)
    t, its = 0.0, 0
    for _ in range(args.steps):
        dt, k = cpu_cfg4_sample(P, per_step)
        t += dt
        its += k
    v = its / t / PROXY_SCALE
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded numpy PCG64 proxy of config 4, reference generator recipe)",
           "config": {"workload": WORKLOAD, "parallelism": "host cores (OpenBLAS threads)",
                      "proxy": "d=8192 n=32768 k=256 fp64 (2 GiB), %d FISTA iterations per step, "
                               "extrapolated x%d by dictionary bytes" % (per_step, PROXY_SCALE)},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                            "sample": "%d steps x %d FISTA iterations on the config-4 proxy"
                                      % (args.steps, per_step)},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------- GPU legs
def stream_roofline(torch, dev):
    """FISTA on a larger-than-L2 dictionary (d=16384, n=65536, fp32 storage =
    4 GiB) for 16 iterations: every panel pass streams A from HBM."""
    from paper_1007_3753_b200 import device as dv
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.shrinkage import FistaPlan
    d, n, k = 16384, 65536, 512
    g = torch.Generator(device=dev)
    g.manual_seed(4)
    A = torch.randn(d, n, device=dev, dtype=torch.float32, generator=g)
    A /= torch.linalg.vector_norm(A, dim=0, keepdim=True)
    x0 = torch.zeros(n, device=dev, dtype=torch.float32)
    idx = torch.randperm(n, device=dev, generator=g)[:k]
    x0[idx] = torch.randn(k, device=dev, generator=g)
    b = (A @ x0).double()
    D = dv.DeviceDictionary(A, dtype="float32", device=dev.index)
    del A
    torch.cuda.empty_cache()

    class _P:
        pass
    P = _P()
    P.A, P.b, P.ground_truth = D, b.cpu().numpy(), None
    P.n, P.d = n, d
    plan = FistaPlan(P, SolverConfig(lam=None, tol=1e-12, max_iter=16,
                                     options={"continuation": False}))
    plan.launch()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    tot = 0.0
    passes = 0.0
    for _ in range(reps):
        s.record()
        plan.launch()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e) / 1e3
        passes += plan.passes()
    bytes_ = passes * d * n * 4
    st = plan.bufs.read_state()
    del plan
    # what shrinkage.fista_solve runs for this dictionary (>= 1 GiB fp32: the
    # streaming route, the sharded rounds at world 1 with the bulk-copy passes)
    from paper_1007_3753_b200 import shrinkage
    from paper_1007_3753_b200.sharded import (DeviceShardOps, ShardedDictionary, ShardedFista,
                                              SoloCollective)
    cfg = SolverConfig(lam=None, tol=1e-12, max_iter=16, options={"continuation": False})
    routed = shrinkage._stream_route(P, cfg, None)
    ops = DeviceShardOps(ShardedDictionary(D, 0, n), SoloCollective())
    bh = P.b
    drv = ShardedFista(ops, bh, n, cfg, b_device=ops.from_host_d(bh))
    drv.solve()
    torch.cuda.synchronize()
    rtot, rpasses, rits = 0.0, 0, 0
    for _ in range(reps):
        s.record()
        r = drv.solve()
        e.record()
        torch.cuda.synchronize()
        rtot += s.elapsed_time(e) / 1e3
        rpasses += drv.passes
        rits += r.iterations
    del drv, ops, D
    torch.cuda.empty_cache()
    return {"shape": "d=16384 n=65536 fp32 storage (4 GiB), 16 FISTA iterations, fixed lambda",
            "kernel": "the persistent single-instance FISTA kernel (FistaPlan, fista.cu)",
            "achieved_gbs": bytes_ / tot / 1e9, "passes_per_launch": passes / reps,
            "ms_per_launch": 1e3 * tot / reps, "iterations": int(st.iterations),
            "fista_solve_route": {"routed": bool(routed),
                                  "path": "sharded rounds at world 1 (gemv / gemv_t_stream passes), what "
                                          "shrinkage.fista_solve takes for >= 1 GiB fp32 dictionaries",
                                  "achieved_gbs": rpasses * d * n * 4 / rtot / 1e9,
                                  "passes_per_solve": rpasses / reps, "iterations": rits // reps,
                                  "ms_per_solve": 1e3 * rtot / reps}}


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _proxy_parity(torch, dev):
    """The config-4 proxy (d=8192, n=32768) through the same sharded path
    against the real reference's output (tests/golden/cfg4_proxy_fista.npz)."""
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200.sharded import ShardedDictionary, ShardedInstance, sharded_fista_solve
    g = np.load(os.path.join(ROOT, "tests", "golden", "cfg4_proxy_fista.npz"))
    rc = json.loads(str(g["recipe"]))
    A = synth.gen_gaussian_dict(rc["d"], rc["n"], rc["seed"])
    out = {}
    for dt in ("float64", "float32"):
        cfg = cfg4_config(5000)
        cfg.options["dtype"] = dt
        shard = ShardedDictionary.from_dense(A, 0, 1, dtype=dt, device_ordinal=dev.index)
        r = sharded_fista_solve(ShardedInstance(shard, g["b"]), cfg)
        ref = g["x"]
        out[dt] = {"rel_err_vs_reference": float(np.linalg.norm(r.x_star - ref) / np.linalg.norm(ref)),
                   "iterations": int(r.iterations), "iterations_reference": int(g["iterations"])}
        del shard
    torch.cuda.empty_cache()
    return out


def headline_cfg4(torch, dev, ws, rank, args):
    from paper_1007_3753_b200 import device as dv
    from paper_1007_3753_b200.sharded import (ShardedFista, ShardedInstance, TorchCollective,
                                              kkt_certificate, make_cfg4_shard, sharded_fista_solve)
    coll = TorchCollective()
    t0 = time.perf_counter()
    shard, b, x0, ops = make_cfg4_shard(rank, ws, dev, coll)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    cfg = cfg4_config()
    b_dev = ops.from_host_d(b)
    drv = ShardedFista(ops, b, shard.n, cfg, b_device=b_dev)
    for _ in range(max(args.warmup, 3)):
        res = drv.solve()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index)
    clocks.start()
    clocks.wait_ready()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    spans, its, passes, rounds, trials = [], 0, 0, 0, 0
    ops.timing = []
    for _ in range(args.steps):
        ev = _events(torch)
        drv.span_events = ev
        res = drv.solve()
        spans.append(ev)
        its += res.iterations
        passes += drv.passes
        rounds += drv.rounds
        trials += drv.trials
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    drv.span_events = None
    timing, ops.timing = ops.timing, None
    tot = sum(s.elapsed_time(e) for s, e in spans) / 1e3
    t_pre = sum(e[0].elapsed_time(e[1]) for e in timing) / 1e3
    t_coll = sum(e[1].elapsed_time(e[2]) for e in timing) / 1e3
    t_post = sum(e[2].elapsed_time(e[3]) for e in timing) / 1e3
    t = torch.tensor([tot, t_pre + t_post], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    tmax, tkern = float(t[0].item()), float(t[1].item())
    value = its / tmax
    # end to end through the public API: host b in (pinned), host x + trace out
    e2e_steps = max(1, min(args.steps, 5))
    b_pin = torch.from_numpy(b).pin_memory().numpy()
    sharded_fista_solve(ShardedInstance(shard, b_pin), cfg, ops=ops)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    es, ee = _events(torch)
    e_its = 0
    es.record()
    for _ in range(e2e_steps):
        r2 = sharded_fista_solve(ShardedInstance(shard, b_pin), cfg, ops=ops)
        e_its += r2.iterations
    ee.record()
    torch.cuda.synchronize()
    ck = clocks.stop()
    te = torch.tensor([es.elapsed_time(ee) / 1e3], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_val = e_its / float(te.item())
    # certificate of the last solution (fp64 recomputation of c = A^T (b - A x))
    lam = 1e-2 * ops.setup(b)
    kk, F = kkt_certificate(ops, res.x_star[shard.c0:shard.c1], b, lam)
    shard_bytes = shard.local.n * shard.d * 4
    alg = passes * shard_bytes
    out = {"value": value, "ms_per_step": 1e3 * tmax / args.steps, "iterations": its,
           "solves_per_sec": args.steps / tmax, "iterations_per_solve": its / args.steps,
           "passes_per_iteration": passes / its, "trials_per_iteration": trials / its,
           "rounds_per_solve": rounds / args.steps, "gen_seconds": gen_s,
           "gpu_launches": args.steps * 5 + 6 * rounds,
           "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(b.nbytes),
                   "d2h_bytes_per_step": int(shard.n * 8 + 32 * res.iterations + 160),
                   "api": "paper_1007_3753_b200.sharded.sharded_fista_solve(ShardedInstance(shard, b), config): "
                          "pinned host b in, host x (n) + trace out; dictionary resident (64 GiB)"},
           "kernel_seconds": {"pre (prox + A_r x)": t_pre, "allreduce": t_coll,
                              "post (decide + A_r^T r + rotate/KKT)": t_post, "step_total": tot},
           "achieved_gbs": alg / tkern / 1e9, "step_gbs": alg / tmax / 1e9,
           "shard_bytes": shard_bytes,
           "certificate": {"kkt_fp64": kk, "lambda": lam, "kkt_over_lambda": kk / lam,
                           "objective": F, "objective_trace": res.trace[-1].objective,
                           "converged": bool(res.converged),
                           "x0_large_entries_recovered": bool(np.all(res.x_star[np.abs(x0) > 4 * lam] != 0))},
           "clocks": ck}
    if ws > 1:
        import torch.distributed as dist
        out["nccl"] = {"backend": dist.get_backend(), "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
    del drv, ops, shard, b_dev
    torch.cuda.empty_cache()
    return out


_PEAKS = {}


def gemm_peaks(torch, dev):
    """Library DGEMM / SGEMM / TF32 throughput on this GPU pool (8192^3): the
    denominators of the batched solvers' tensor-pipe roofline (only bf16 is in
    MEASURED_PEAKS.json).  Read from profiles/r02_gemm_peaks.json
    (tools/gemm_peaks.py, measured on this pool) so the bench launches no
    library kernels; measured here only when that file is missing."""
    if _PEAKS:
        return _PEAKS
    path = os.path.join(ROOT, "profiles", "r02_gemm_peaks.json")
    if os.path.exists(path):
        try:
            _PEAKS.update(json.load(open(path)))
            if all(k in _PEAKS for k in ("dgemm_tflops", "sgemm_tflops", "tf32_tflops")):
                return _PEAKS
        except ValueError:
            _PEAKS.clear()
    for name, dt in (("dgemm_tflops", torch.float64), ("sgemm_tflops", torch.float32)):
        a = torch.randn(8192, 8192, device=dev, dtype=dt)
        b = torch.randn(8192, 8192, device=dev, dtype=dt)
        torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            s, e = _events(torch)
            s.record()
            torch.matmul(a, b)
            e.record()
            torch.cuda.synchronize()
            best = max(best, 2 * 8192 ** 3 / (s.elapsed_time(e) / 1e3) / 1e12)
        _PEAKS[name] = best
        del a, b
    # dense TF32 tensor-pipe throughput (cuBLAS, fp32 operands with TF32 math)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn(8192, 8192, device=dev, dtype=torch.float32)
        b = torch.randn(8192, 8192, device=dev, dtype=torch.float32)
        torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            s, e = _events(torch)
            s.record()
            torch.matmul(a, b)
            e.record()
            torch.cuda.synchronize()
            best = max(best, 2 * 8192 ** 3 / (s.elapsed_time(e) / 1e3) / 1e12)
        _PEAKS["tf32_tflops"] = best
        del a, b
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    torch.cuda.empty_cache()
    return _PEAKS


def leg_cfg3(torch, dev, queries=1024):
    """BASELINE config 3: CAB [A I] (d=1024, 38 classes x 32 columns), 1024
    corrupted queries, batched dual ALM in fp32 storage + SRC labels."""
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200.batched import src_classify
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.robust import ExtendedDictionary
    A, lab = synth.cab_dictionary(d=1024, classes=38, per_class=32, subspace=9, seed=0)
    Bq, truth = synth.cab_queries(A, lab, queries, fraction=0.2, seed=1)
    cfg = SolverConfig(tol=1e-4, max_iter=2000, options={"dtype": "float32"})
    ext = ExtendedDictionary(A, 1.0, dtype="float32", device_ordinal=dev.index)
    Bmat = np.ascontiguousarray(Bq.T)
    src_classify(ext, lab, Bmat, cfg)             # warm-up (Gram factor cached)
    torch.cuda.synchronize()
    s, e = _events(torch)
    s.record()
    labels, _, res = src_classify(ext, lab, Bmat, cfg)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 1e3
    its = res.iterations.astype(np.int64)
    # 2 passes over A (4 d n_A) + the two triangular solves with the
    # row-Gram factor (2 d^2) per query-iteration (7.08 MFLOP; 7.25 GFLOP per
    # batched iteration at 1024 queries); the identity block costs nothing
    d_, nA = 1024, 1216
    tfl = float(its.sum()) * (4.0 * d_ * nA + 2.0 * d_ * d_) / t / 1e12
    exec_per = 2.0 * d_ * (nA + d_) + 2.0 * d_ * nA + 2.0 * nA * d_ + 4.0 * d_ * nA
    tfl_exec = float(its.sum()) * exec_per / t / 1e12
    peaks = gemm_peaks(torch, dev)
    return {"workload": "cfg3: CAB [A I] 1024 x 2240, %d queries, batched DALM fp32 storage, "
                        "tol 1e-4, min-class-residual labels" % queries,
            "roofline": {"bound": "tensor (3xTF32 tcgen05)", "achieved": 3 * tfl, "peak": peaks["tf32_tflops"],
                         "unit": "TFLOP/s", "frac": 3 * tfl / peaks["tf32_tflops"],
                         "peak_source": "cuBLAS TF32 8192^3 (profiles/r02_gemm_peaks.json)",
                         "algorithmic": "SURVEY 8(d): (4 d n_A + 2 d^2) flops per query-iteration, x3 TF32 "
                                        "MMAs per fp32-accurate product",
                         "fp32_accurate_tflops": tfl,
                         # the products the batched iteration actually runs (batch_dalm.cu main_part /
                         # tail_part, fp32 [A, sI]): [M | Ginv] V (K = n_A + d), A Z, A^T Y, A [U | x_new]
                         "executed_mma_tflops": 3 * tfl_exec,
                         "executed_frac": 3 * tfl_exec / peaks["tf32_tflops"],
                         "executed": "2 d (n_A + d) + 2 d n_A + 2 n_A d + 4 d n_A = %.2f MFLOP per "
                                     "query-iteration (x3 MMAs)" % (exec_per / 1e6),
                         # frac can reach at most algorithmic / executed flops: the iteration also forms
                         # the reference's y-step certificate A A^T y and the residual b - A x (alm.py:181,
                         # 249), which SURVEY 8(d) does not count
                         "ceiling_frac": (4.0 * d_ * nA + 2.0 * d_ * d_) / exec_per,
                         "gemm_share_of_batch": "57% of the kernel time is in the GEMMs, whose main loops run "
                                                "at 90-95% of the tf32 MMA rate (DESIGN 3.4.1)"},
            "queries_per_sec": queries / t, "ms_per_batch": 1e3 * t,
            "mean_iterations": float(its.mean()), "max_iterations": int(its.max()),
            "accuracy_vs_truth": float(np.mean(labels == truth)),
            "fp32_gemm": "3xTF32 tcgen05 kernel (tc_gemm.cu)",
            "note": "timed through the public call (host queries in, labels out)",
            "cpu_baseline": cpu_pool_rate("cab_dalm", A, [Bq[q] for q in range(queries)], per_core=4)}


def leg_cfg5(torch, dev, ws=1, B=1024, cpu_sample=4):
    """BASELINE config 5 point: B instances sharing one A (512 x 2048, fp64),
    k ~ U[16, 256], noiseless b = A x0; batched FISTA (lambda 1e-3,
    relative-estimate 1e-6), batched dual ALM (relative-estimate 1e-6) and
    batched Homotopy (target lambda 1e-3).  N > 1: instances dealt
    round-robin across the ranks (A replicated, no per-iteration
    communication), time = max over ranks (strong scaling, B fixed)."""
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200 import device as dv
    from paper_1007_3753_b200.batched import dalm_solve_batch, fista_solve_batch, homotopy_solve_batch
    from paper_1007_3753_b200.distributed import solve_batch_sharded
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    d, n = 512, 2048
    A, _, Bmat = synth.cfg5_batch(B)
    D = dv.DeviceDictionary(A, dtype="float64", device=dev.index)
    rel = StoppingRule("relative-estimate", 1e-6)
    legs = {
        "fista": (fista_solve_batch, SolverConfig(lam=1e-3, tol=1e-6, max_iter=5000, stopping=rel), {}),
        "dalm": (dalm_solve_batch, SolverConfig(tol=1e-6, max_iter=5000, stopping=rel), {}),
        "homotopy": (homotopy_solve_batch, SolverConfig(max_iter=5000), {"target_lambda": 1e-3}),
    }
    out = {"workload": "cfg5: B=%d instances, shared A 512 x 2048 fp64, k~U[16,256], noiseless" % B,
           "n_gpus": ws, "scaling": "strong (B fixed, instances dealt across ranks)",
           "note": "timed through the public call (host B in, host X out), max over ranks"}
    for name, (fn, cfg, kw) in legs.items():
        def run(Bm, fn=fn, cfg=cfg, kw=kw):
            if "target_lambda" in kw:
                return solve_batch_sharded(lambda A_, B_, c_: fn(A_, B_, kw["target_lambda"], c_), D, Bm, cfg)
            return solve_batch_sharded(fn, D, Bm, cfg)
        run(Bmat[:, : 16 * ws])                     # warm-up (Gram factor, cuBLAS handles)
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        s, e = _events(torch)
        s.record()
        res = run(Bmat)
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / 1e3], dtype=torch.float64, device=dev)
        if ws > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t = float(t.item())
        its = res.iterations.astype(np.int64)
        unit = "breakpoints_per_sec" if name == "homotopy" else "iterations_per_sec"
        # SURVEY §8(d) algorithmic flops per instance-iteration: FISTA 2 passes (4 d n),
        # DALM 2 passes + 2 triangular solves (4 d n + 2 d^2), Homotopy the 2 A^T passes (4 d n)
        per = {"fista": 4.0 * d * n, "dalm": 4.0 * d * n + 2.0 * d * d, "homotopy": 4.0 * d * n}[name]
        tfl = float(its.sum()) * per / t / 1e12
        pk = gemm_peaks(torch, dev)["dgemm_tflops"]
        out[name] = {"solves_per_sec": B / t, "ms_per_batch": 1e3 * t, unit: float(its.sum()) / t,
                     "mean_iterations": float(its.mean()), "converged": int(res.converged.sum()),
                     "roofline": {"bound": "tensor (fp64 DMMA GEMMs)", "achieved": tfl,
                                  "peak": pk, "unit": "TFLOP/s", "frac": tfl / pk,
                                  "peak_source": "cuBLAS DGEMM 8192^3 (profiles/r02_gemm_peaks.json)",
                                  "algorithmic": {"fista": "4 d n", "dalm": "4 d n + 2 d^2",
                                                  "homotopy": "4 d n (the two A^T passes)"}[name]
                                                 + " flops per instance-iteration (SURVEY 8(d))"}}
    if ws == 1 and cpu_sample > 0:
        # CPU reference port on a bounded sample of the same instances (all host cores, process pool)
        cols = [Bmat[:, j] for j in range(B)]
        out["cpu_baseline"] = {name: cpu_pool_rate(name, A, cols, per_core=cpu_sample)
                               for name in ("fista", "homotopy", "dalm")}
    return out


def leg_cfg1(torch, reps=5):
    """BASELINE config 1 (configs[0], the reference's CPU-runnable case):
    d=500, n=1000, k=50 noiseless, fp64; FISTA / PALM / DALM at lambda 1e-3,
    relative change in x < 1e-6; solves/s next to the CPU port."""
    from paper_1007_3753_b200 import device as dv, synth
    from paper_1007_3753_b200.alm import dalm_solve, palm_solve
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig, StoppingRule
    from paper_1007_3753_b200.shrinkage import fista_solve
    import oracle
    P = synth.make_problem(synth.CFG1)
    D = dv.DeviceDictionary(P.A)
    Pd = ProblemInstance.__new__(ProblemInstance)
    Pd.A, Pd.b, Pd.ground_truth, Pd.noise_sigma = D, P.b, P.ground_truth, P.noise_sigma
    rel = StoppingRule("relative-estimate", 1e-6)
    out = {"workload": "cfg1: d=500 n=1000 k=50 noiseless fp64, lambda 1e-3, relative change in x < 1e-6"}
    legs = {"fista": (lambda: fista_solve(Pd, SolverConfig(lam=1e-3, tol=1e-6, stopping=rel)),
                      lambda: oracle.fista(P.A, P.b, lam=1e-3, tol=1e-6, stop=("relative-estimate", 1e-6))),
            "palm": (lambda: palm_solve(Pd, SolverConfig(tol=1e-6, stopping=rel)),
                     lambda: oracle.palm(P.A, P.b, tol=1e-6, stop=("relative-estimate", 1e-6))),
            "dalm": (lambda: dalm_solve(Pd, SolverConfig(tol=1e-6, stopping=rel)),
                     lambda: oracle.dalm(P.A, P.b, tol=1e-6, stop=("relative-estimate", 1e-6)))}
    for name, (gpu, cpu) in legs.items():
        r = gpu()
        torch.cuda.synchronize()
        s, e = _events(torch)
        s.record()
        for _ in range(reps):
            r = gpu()
        e.record()
        torch.cuda.synchronize()
        t = s.elapsed_time(e) / 1e3 / reps
        t0 = time.perf_counter()
        rc = cpu()
        tc = time.perf_counter() - t0
        err = float(np.linalg.norm(r.x_star - rc.x) / max(np.linalg.norm(rc.x), 1e-300))
        out[name] = {"solves_per_sec": 1.0 / t, "ms_per_solve": 1e3 * t, "iterations": int(r.iterations),
                     "cpu_port_solves_per_sec": 1.0 / tc, "cpu_iterations": int(rc.iterations),
                     "rel_err_vs_oracle": err}
    out["cpu_cores"] = os.cpu_count()
    return out


def leg_cfg5_sweep(torch, dev, sizes=(1, 16, 256, 1024, 8192), homotopy=True):
    """BASELINE config 5 batch-size sweep (FISTA fp64 and fp32, Homotopy fp64)."""
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200 import device as dv
    from paper_1007_3753_b200.batched import fista_solve_batch, homotopy_solve_batch
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    d, n = 512, 2048
    A, _, Bmat = synth.cfg5_batch(max(sizes))
    rel = StoppingRule("relative-estimate", 1e-6)
    D64 = dv.DeviceDictionary(A, dtype="float64", device=dev.index)
    D32 = dv.DeviceDictionary(A, dtype="float32", device=dev.index)
    rows = []
    if min(sizes) > 16:                                  # one-time setup (operand splits, graphs) outside the timings
        for D_ in (D64, D32):
            fista_solve_batch(D_, np.ascontiguousarray(Bmat[:, :16]), SolverConfig(lam=1e-3, stopping=rel))
    for B in sizes:
        row = {"B": B}
        for name, fn in (("fista_f64", lambda Bm: fista_solve_batch(D64, Bm, SolverConfig(lam=1e-3, stopping=rel))),
                         ("fista_f32", lambda Bm: fista_solve_batch(D32, Bm, SolverConfig(lam=1e-3, stopping=rel))),
                         ("homotopy_f64", lambda Bm: homotopy_solve_batch(D64, Bm, 1e-3, SolverConfig()))):
            if name == "homotopy_f64" and not homotopy:
                continue
            s, e = _events(torch)
            torch.cuda.synchronize()
            s.record()
            r = fn(np.ascontiguousarray(Bmat[:, :B]))
            e.record()
            torch.cuda.synchronize()
            t = s.elapsed_time(e) / 1e3
            row[name] = {"solves_per_sec": B / t, "iterations_per_sec": float(r.iterations.sum()) / t}
            # SURVEY 8(d) tensor fraction: 4 d n flops per instance-iteration (both products of an
            # iteration), x3 TF32 MMAs per fp32-accurate product, against the library peak of the pipe
            tfl = float(r.iterations.sum()) * 4.0 * d * n / t / 1e12
            pk = gemm_peaks(torch, dev)
            if name == "fista_f32":
                row[name]["tensor_frac"] = 3.0 * tfl / pk["tf32_tflops"]
            else:
                row[name]["tensor_frac"] = tfl / pk["dgemm_tflops"]
        rows.append(row)
    return {"workload": "cfg5 sweep: shared A 512 x 2048, k~U[16,256], lambda 1e-3", "rows": rows,
            "tensor_frac": "4 d n flops per instance-iteration (SURVEY 8(d)); fp32 x3 (3xTF32 MMAs) over the "
                           "cuBLAS TF32 peak, fp64 over the cuBLAS DGEMM peak (profiles/r02_gemm_peaks.json)"}


def leg_align(torch, count=4096, d=1024, m=11, cpu_sample=64):
    """PALM alignment (robust.py:470-515) batched across
    images — `count` images of d pixels, m parameters, 20% grossly corrupted
    rows — vs the numpy restatement (oracle.align_palm) on host cores."""
    from paper_1007_3753_b200 import robust
    from paper_1007_3753_b200.model import SolverConfig
    from tests.golden.align_cases import align_instance
    insts = [align_instance(seed=1000 + j, d=d, m=m, frac=0.2) for j in range(count)]
    Bs = np.stack([B for B, _ in insts])
    bs = np.stack([b for _, b in insts])
    cfg = SolverConfig(tol=1e-8, max_iter=5000)
    robust.align_palm_solve_batch(Bs[:64], bs[:64], cfg)       # warm-up
    torch.cuda.synchronize()
    s, e = _events(torch)
    s.record()
    W, E = robust.align_palm_solve_batch(Bs, bs, cfg)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 1e3
    # the same batch with the images already resident (device throughput of the kernel)
    Bd = torch.from_numpy(Bs).cuda()
    bd = torch.from_numpy(bs).cuda()
    robust.align_batch_device("palm", Bd[:64], bd[:64], cfg)
    torch.cuda.synchronize()
    s2, e2 = _events(torch)
    s2.record()
    W2, _, its = robust.align_batch_device("palm", Bd, bd, cfg)
    e2.record()
    torch.cuda.synchronize()
    td = s2.elapsed_time(e2) / 1e3
    its = its.cpu().numpy()
    from oracle.l1_oracle import align_palm
    worst = 0.0
    for j in range(8):                                    # parity spot check against the port
        w_ref, e_ref = align_palm(Bs[j], bs[j], tol=1e-8, max_iter=5000)
        worst = max(worst, float(np.linalg.norm(W[j] - w_ref) / np.linalg.norm(w_ref)))
    ncpu = min(count, cpu_sample * os.cpu_count())
    rate, _, tc, cores = cpu_pool_tasks([("align_palm", Bs[j], bs[j]) for j in range(ncpu)])
    return {"workload": "PALM alignment, %d images, d=%d pixels, m=%d parameters, 20%% corrupted rows, "
                        "tol 1e-8 (public call: host images in, host w/e out)" % (count, d, m),
            "images_per_sec": count / t, "ms_per_batch": 1e3 * t,
            "device_images_per_sec": count / td, "device_ms_per_batch": 1e3 * td,
            "mean_palm_steps": float(its.mean()),
            "bitwise_equal_resident_vs_host_call": bool(np.array_equal(W2.cpu().numpy(), W)),
            "cpu_port_images_per_sec": rate,
            "cpu_sample": "first %d images, ProcessPoolExecutor(%d warm workers, 1 BLAS thread each), %.1f s"
                          % (ncpu, cores, tc),
            "max_rel_err_w_vs_port": worst}


def leg_harness(torch, n=200, grid=10, trials=10, cpu_sample=8):
    """the experiment harness on the GPU.  A phase grid
    (bench.run_phase_grid: rho x delta = grid x grid cells, `trials` fresh
    instances each, one dictionary per trial, tol 1e-8, max_iter 20000,
    lambda 1e-4 ||A^T b||_inf) solved in group launches, plus the reference
    acceptance suite's noise sweep (criterion 5).  Timed: device solve of
    all trials (dictionaries already uploaded) and the whole harness call
    (host instances in, success rates out)."""
    from paper_1007_3753_b200 import harness
    from paper_1007_3753_b200.group import TrialGroup
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.synth import GenSpec, make_instance, trial_seed
    rhos = [round(0.02 + 0.38 * i / (grid - 1), 4) for i in range(grid)]
    deltas = [round(0.1 + 0.9 * j / (grid - 1), 4) for j in range(grid)]
    probs = []
    for i, rho in enumerate(rhos):
        for j, delta in enumerate(deltas):
            k, d = max(1, int(round(rho * n))), max(1, int(round(delta * n)))
            for t in range(trials):
                probs.append(make_instance(GenSpec(n=n, d=d, k=k, seed=trial_seed(0, i, j, t))))
    out = {"workload": "phase grid n=%d, %dx%d cells (rho %.2f..%.2f, delta %.2f..%.2f), %d trials/cell = %d "
                       "trials, one Gaussian dictionary per trial, tol 1e-8, lambda 1e-4||A^T b||_inf"
                       % (n, grid, grid, rhos[0], rhos[-1], deltas[0], deltas[-1], trials, len(probs))}
    cfg = SolverConfig(tol=1e-8, max_iter=20000)
    for name in ("fista", "homotopy", "dalm"):
        grp = TrialGroup(probs)
        lams = 1e-4 * grp.correlation_max()
        grp.solve(name, SolverConfig(tol=1e-8, max_iter=5), lams=lams)        # warm-up (module load)
        torch.cuda.synchronize()
        s, e = _events(torch)
        s.record()
        res = grp.solve(name, cfg, lams=lams)
        e.record()
        torch.cuda.synchronize()
        sec = s.elapsed_time(e) / 1e3
        its = np.array([r.iterations for r in res])
        ok = np.mean([np.linalg.norm(r.x_star - P.ground_truth) <= 1e-3 * np.linalg.norm(P.ground_truth)
                      for r, P in zip(res, probs)])
        t0 = time.perf_counter()
        harness.run_phase_grid(name, n, rhos, deltas, trials)
        whole = time.perf_counter() - t0
        out[name] = {"trials_per_sec": len(probs) / sec, "device_seconds": sec,
                     "harness_call_seconds": whole, "mean_iterations": float(its.mean()),
                     "max_iterations": int(its.max()), "success_fraction": float(ok)}
    # CPU port (the reference's per-trial solve) over a process pool of all host
    # cores — the reference harness fans trials over processes the same way
    cpu = {}
    ncpu = min(len(probs), cpu_sample * os.cpu_count())
    sample = probs[:: max(1, len(probs) // ncpu)][:ncpu]
    for name in ("fista", "homotopy", "dalm"):
        tasks = [("harness_" + name, P.A, P.b, 1e-4 * float(np.max(np.abs(P.A.T @ P.b)))) for P in sample]
        rate, _, el, cores = cpu_pool_tasks(tasks)
        cpu[name + "_trials_per_sec"] = rate
    cpu.update({"cores": os.cpu_count(), "kind": "port",
                "sample": "%d trials spread over the grid per solver, ProcessPoolExecutor(%d workers, 1 BLAS "
                          "thread each)" % (len(sample), os.cpu_count())})
    out["cpu_baseline"] = cpu
    # acceptance criterion 5 noise sweep (test_acceptance.py:128-160), jobs ignored
    t0 = time.perf_counter()
    sw = harness.run_noise_sweep(("homotopy", "gpsr", "tnipm", "ist", "fista"), "vary-d",
                                 {"n": 400, "k": 40, "d_values": [160, 200, 240, 280, 320, 360, 380],
                                  "noise_sigma": 0.01}, trials=20, base_seed=0)
    out["noise_sweep_criterion5"] = {"seconds": time.perf_counter() - t0,
                                     "final_rel_error": {s: float(sw.mean_rel_error[q, -1])
                                                         for q, s in enumerate(sw.solvers)},
                                     "reference_bound_seconds": 300.0,
                                     "note": "7 d values x 20 trials x 5 solvers, one call"}
    return out


def leg_solvers_cfg2(torch, P, reps=3):
    """Every single-instance solver on the cfg2 instance (ms per solve)."""
    from paper_1007_3753_b200 import device as dv
    from paper_1007_3753_b200.alm import dalm_solve, palm_solve
    from paper_1007_3753_b200.gradient_projection import gpsr_solve, tnipm_solve
    from paper_1007_3753_b200.homotopy import homotopy_solve
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig, StoppingRule
    from paper_1007_3753_b200.pdipa import pdipa_solve
    from paper_1007_3753_b200.shrinkage import fista_solve, ist_solve
    D = dv.DeviceDictionary(P.A)
    Pd = ProblemInstance.__new__(ProblemInstance)
    Pd.A, Pd.b, Pd.ground_truth, Pd.noise_sigma = D, P.b, P.ground_truth, P.noise_sigma
    lam = 1e-2 * float(np.max(np.abs(P.A.T @ P.b)))
    rel = StoppingRule("relative-estimate", 1e-6)
    cfg = SolverConfig(lam=None, tol=1e-6, stopping=rel)
    cfgl = SolverConfig(lam=lam, tol=1e-6, stopping=rel)
    runs = {"fista": lambda: fista_solve(Pd, cfg),
            "ist": lambda: ist_solve(Pd, None, cfg),
            "palm": lambda: palm_solve(Pd, cfg),
            "dalm": lambda: dalm_solve(Pd, cfg),
            "gpsr": lambda: gpsr_solve(Pd, lam, cfgl),
            "tnipm": lambda: tnipm_solve(Pd, lam, cfgl),
            "homotopy": lambda: homotopy_solve(Pd, lam, SolverConfig()),
            "pdipa": lambda: pdipa_solve(Pd, SolverConfig(tol=1e-6))}
    out = {}
    for name, fn in runs.items():
        try:
            fn()
            torch.cuda.synchronize()
            s, e = _events(torch)
            s.record()
            for _ in range(reps):
                r = fn()
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / reps
            out[name] = {"ms_per_solve": round(ms, 3), "iterations": int(r.iterations),
                         "converged": bool(r.converged),
                         "us_per_iteration": round(1e3 * ms / max(int(r.iterations), 1), 2)}
        except Exception as exc:  # pragma: no cover - report, do not abort the bench
            out[name] = {"error": str(exc)[:160]}
    # CPU port: the same solvers for a bounded number of iterations (per-iteration rate)
    import oracle
    cap = 40
    cpu = {"fista": lambda: oracle.fista(P.A, P.b, tol=1e-6, max_iter=cap),
           "ist": lambda: oracle.ist(P.A, P.b, lam=lam, tol=1e-6, max_iter=cap),
           "palm": lambda: oracle.palm(P.A, P.b, tol=1e-6, max_iter=cap),
           "dalm": lambda: oracle.dalm(P.A, P.b, tol=1e-6, max_iter=cap),
           "gpsr": lambda: oracle.gpsr(P.A, P.b, lam=lam, tol=1e-6, max_iter=cap),
           "tnipm": lambda: oracle.tnipm(P.A, P.b, lam=lam, tol=1e-6, max_iter=8),
           "homotopy": lambda: oracle.homotopy(P.A, P.b, lam, max_iter=cap)[0],
           "pdipa": lambda: oracle.pdipa(P.A, P.b, tol=1e-6, max_iter=8)}
    for name, fn in cpu.items():
        try:
            t0 = time.perf_counter()
            r = fn()
            el = time.perf_counter() - t0
            if name in out and isinstance(out[name], dict):
                out[name]["cpu_port_us_per_iteration"] = round(1e6 * el / max(int(r.iterations), 1), 1)
        except Exception as exc:  # pragma: no cover
            if name in out and isinstance(out[name], dict):
                out[name]["cpu_port_error"] = str(exc)[:120]
    out["cpu_note"] = ("cpu_port_us_per_iteration: oracle port (numpy/OpenBLAS, %d host cores) run for "
                       "a bounded number of iterations on the same instance" % os.cpu_count())
    return out


def leg_cfg2(torch, dev, steps=20, warmup=3, dtype="float64"):
    """BASELINE config 2 (configs[1]): one complete FISTA solve per step on the
    resident 32 MiB dictionary (SMEM/L2-resident after the first pass: the
    single persistent kernel is latency-bound, reported against HBM for
    reference only), plus its end-to-end public call and the CPU port."""
    from paper_1007_3753_b200 import device as dv
    from paper_1007_3753_b200.model import ProblemInstance
    from paper_1007_3753_b200.shrinkage import FistaPlan, fista_solve
    import oracle  # checker: parity of the timed solve
    P = make_instance(0)
    cfg = config(dtype)
    D = dv.DeviceDictionary(P.A, dtype=dtype, device=dev.index)
    Pd = ProblemInstance.__new__(ProblemInstance)
    Pd.A, Pd.b, Pd.ground_truth, Pd.noise_sigma = D, P.b, P.ground_truth, P.noise_sigma
    plan = FistaPlan(Pd, cfg)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # 512 MiB > L2
    for _ in range(max(warmup, 3)):
        plan.launch()
    torch.cuda.synchronize()
    res = plan.result()
    iters = res.iterations
    passes = plan.passes()
    ev = [_events(torch) for _ in range(steps)]
    torch.cuda.synchronize()
    for s, e in ev:
        flush.zero_()                      # evict A from L2 between timed steps
        s.record()
        plan.launch()
        e.record()
    torch.cuda.synchronize()
    tot = sum(s.elapsed_time(e) for s, e in ev) / 1e3
    e2e_steps = 5
    pin_A = torch.from_numpy(P.A).pin_memory()
    pin_b = torch.from_numpy(P.b).pin_memory()
    Ph = ProblemInstance(pin_A.numpy(), pin_b.numpy(), ground_truth=P.ground_truth)
    fista_solve(Ph, cfg)
    torch.cuda.synchronize()
    es, ee = _events(torch)
    es.record()
    for _ in range(e2e_steps):
        r = fista_solve(Ph, cfg)
    ee.record()
    torch.cuda.synchronize()
    e2e_val = e2e_steps / (es.elapsed_time(ee) / 1e3)
    ref = cpu_solve_once(P)
    err = float(np.linalg.norm(res.x_star - ref.x) / np.linalg.norm(ref.x))
    sz = 8 if dtype == "float64" else 4
    alg = passes * P.d * P.n * sz
    t1 = tot / steps
    del flush, plan, D
    torch.cuda.empty_cache()
    return {"workload": CFG2_WORKLOAD, "solves_per_sec": steps / tot, "ms_per_solve": 1e3 * t1,
            "iterations_per_solve": iters, "us_per_iteration": 1e6 * t1 / iters,
            "parity": {"rel_err_vs_oracle": err, "iterations_oracle": ref.iterations, "iterations_b200": iters},
            "e2e": {"value": e2e_val, "unit": "solves/s", "h2d_bytes_per_step": int(P.A.nbytes + P.b.nbytes),
                    "d2h_bytes_per_step": int(P.n * 8 + 32 * r.iterations + 256),
                    "api": "shrinkage.fista_solve(P, config), pinned host A/b"},
            "roofline_l2": {"bound": "latency (A 32 MiB is SMEM/L2-resident after the first pass)",
                            "dictionary_bytes_per_second": alg / t1 / 1e9, "unit": "GB/s",
                            "passes_per_solve": passes,
                            "note": "2 grid barriers + region reductions per iteration; see profiles/"},
            "cpu_baseline": cpu_baseline_cfg2(P)}


def run_b200(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    if args.only_leg:
        legs = {"harness": lambda: leg_harness(torch), "cfg1": lambda: leg_cfg1(torch),
                "align": lambda: leg_align(torch), "cfg2": lambda: leg_cfg2(torch, dev),
                "cfg3": lambda: leg_cfg3(torch, dev), "cfg5": lambda: leg_cfg5(torch, dev, ws),
                "cfg5_sweep": lambda: leg_cfg5_sweep(torch, dev),
                "solvers_cfg2": lambda: leg_solvers_cfg2(torch, make_instance(rank)),
                "cfg4": lambda: headline_cfg4(torch, dev, ws, rank, args),
                "stream": lambda: stream_roofline(torch, dev),
                "proxy": lambda: _proxy_parity(torch, dev)}
        r = legs[args.only_leg]()
        if rank == 0:
            print(json.dumps({args.only_leg: r}), flush=True)
        return

    h = headline_cfg4(torch, dev, ws, rank, args)
    out = None
    if rank == 0:
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {}
        peak = float(peaks.get("hbm_gbs", 6650.0))
        traffic = None
        prof = os.path.join(ROOT, "profiles", "r02_ncu_cfg4_full.json")
        if os.path.exists(prof):
            try:
                # ncu dram read+write per pass over the whole 64 GiB dictionary, scaled to this run's shard
                traffic = json.load(open(prof))["traffic_over_algorithmic"] * h["shard_bytes"]
            except (ValueError, KeyError):
                traffic = None
        out = {"metric": METRIC, "value": h["value"], "unit": UNIT, "n_gpus": ws,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": h["ms_per_step"],
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f32 storage / f64 accumulate",
               "data": "synthetic (device Philox dictionary per 2048-column chunk, numpy PCG64 x0/noise)",
               "config": {"workload": WORKLOAD, "solver": "fista",
                          "parallelism": "column-sharded over %d GPU(s), one NCCL allreduce per trial" % ws
                          if ws > 1 else "single GPU (whole 64 GiB dictionary)",
                          "l2": "inputs larger than L2 (64 GiB dictionary >> 126 MB L2); no flush needed"},
               "solves_per_sec": h["solves_per_sec"], "iterations_per_solve": h["iterations_per_solve"],
               "gpu_launches": h["gpu_launches"],
               "e2e": h["e2e"],
               "roofline": {"bound": "hbm", "achieved": h["achieved_gbs"], "peak": peak, "unit": "GB/s",
                            "frac": h["achieved_gbs"] / peak, "traffic": traffic,
                            "kernel": "the two dictionary passes: gemv_stream_kernel (A_r x partials + the "
                                      "fixed-order row reduction) and gemv_t_stream_kernel (A_r^T r), with the "
                                      "elementwise round kernels",
                            "algorithmic": "d * n_local * 4 bytes per pass (%d bytes); passes = 1 A_r x per "
                                           "trial + 1 A_r^T r per accepted iteration; time = CUDA events "
                                           "around ell1_sfista_pre + ell1_sfista_post of every timed round "
                                           "(collective excluded)" % h["shard_bytes"],
                            "step_gbs": h["step_gbs"],
                            "traffic_source": "profiles/r02_ncu_cfg4_full.json: dram__bytes_read.sum + "
                                              "dram__bytes_write.sum per pass (mean of the two passes) / "
                                              "algorithmic bytes, x this run's bytes per pass",
                            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, read+write); the passes are "
                                           "read-only streams, which run slightly above a copy (frac can "
                                           "exceed 1: 7.0 TB/s for one 64 GiB read pass alone, "
                                           "tools/gemv_bench.py --full)"
                            if "hbm_gbs" in peaks else "fallback"},
               "headline_detail": {k: h[k] for k in ("iterations", "passes_per_iteration", "trials_per_iteration",
                                                      "rounds_per_solve", "kernel_seconds", "gen_seconds",
                                                      "certificate") if k in h},
               "clocks": h["clocks"]}
        if "nccl" in h:
            out["nccl"] = h["nccl"]
        if ws == 1:
            try:
                out["parity"] = {"cfg4_proxy_vs_reference": _proxy_parity(torch, dev),
                                 "cfg4_full_scale_certificate": h["certificate"]}
            except Exception as exc:  # pragma: no cover - report, do not abort the bench
                out["parity"] = {"error": str(exc)[:200]}
        if not args.no_stream and ws == 1:
            try:
                rs = stream_roofline(torch, dev)
                rs["frac"] = rs["achieved_gbs"] / peak
                rs["peak"] = peak
                rs["fista_solve_route"]["frac"] = rs["fista_solve_route"]["achieved_gbs"] / peak
                out["roofline_stream"] = rs
            except Exception as exc:  # pragma: no cover - best effort leg
                out["roofline_stream"] = {"error": str(exc)[:200]}
        if not args.no_secondary and ws == 1:
            sec = {}
            legs2 = [("cfg2", lambda: leg_cfg2(torch, dev)), ("cfg1", lambda: leg_cfg1(torch))]
            if args.cfg5_sweep:
                legs2.append(("cfg5_sweep", lambda: leg_cfg5_sweep(torch, dev)))
            else:                   # the large-batch end of the sweep (FISTA fp64 / fp32), ~15 s
                legs2.append(("cfg5_sweep", lambda: leg_cfg5_sweep(torch, dev, sizes=(8192,), homotopy=False)))
            legs2 += [("solvers_cfg2", lambda: leg_solvers_cfg2(torch, make_instance(0))),
                      ("cfg3", lambda: leg_cfg3(torch, dev)),
                      ("cfg5", lambda: leg_cfg5(torch, dev, ws)),
                      ("harness", lambda: leg_harness(torch)),
                      ("align", lambda: leg_align(torch))]
            for name, fn in legs2:
                try:
                    sec[name] = fn()
                except Exception as exc:  # pragma: no cover - best effort leg
                    sec[name] = {"error": str(exc)[:200]}
            out["secondary"] = sec
        if ws == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_cfg4()
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


def run_dry(args):
    """CPU dry run (no GPU): the launcher, a gloo rendezvous and the sharded
    control protocol (numpy restatement of the device rounds, one allreduce
    per round) on the config-1-sized proxy; prints the bench line shape with
    n_gpus = world size.  Not a measurement."""
    import torch.distributed as dist
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200.sharded import ShardedFista, column_range
    from tests.shard_numpy_ops import NumpyShardOps
    P = synth.make_problem(synth.Workload("dry", 500, 1000, 50, seed=0, noise_rel=1e-3))
    c0, c1 = column_range(P.n, rank, ws)
    drv = ShardedFista(NumpyShardOps(P.A[:, c0:c1], P.n), P.b, P.n, cfg4_config())
    t0 = time.perf_counter()
    res = drv.solve()
    el = time.perf_counter() - t0
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": ws, "dry_run": True,
                          "backend": "gloo" if ws > 1 else "none", "iterations": res.iterations,
                          "rounds": drv.rounds, "converged": bool(res.converged), "seconds": el,
                          "note": "CPU dry run of the launcher and the one-allreduce-per-round protocol "
                                  "(d=500 n=1000 proxy, numpy shard ops); no timing claim"}), flush=True)


def main():
    args = parse()
    rc = maybe_launch(args)
    if rc is not None:
        sys.exit(rc)
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
