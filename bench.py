"""Benchmark: H2* / (H2+H)* matvec on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--variants h2star-bt,h2plusH-star]

Workload (configs[1]): 2D, N = 1,048,576 points i.i.d. uniform in [-1,1]^2
(seed 42, reference bench.py:41), K(x,y) = log|x-y| (Log2D, kernels.py:63-71),
quadtree leaf <= 64, NCA tolerance 1e-8, single RHS q ~ N(0,1) (seed 43).  The
operator is built on the box by the native builder (libh2b.so), which
restates the reference construction (identical ranks/pivots on every golden
case); the reference's own Python build is infeasible here (~30 min).

A step is one matvec phi = K~ q.  ``value`` = matvecs/s of the headline
variant (h2star-bt) over all ranks, device-timed with CUDA events on the
plan's stream, inputs resident in HBM; the operator (6.6 GB) is far larger
than L2 (126 MB), so no flush is needed.  ``e2e`` is the same metric through
the public API (GpuHierRep.matvec(q, out=phi) on pinned host vectors: H2D
copy, matvec, D2H copy inside the timed region).  ``roofline`` reports the streaming GEMV
kernel's achieved algorithmic bytes/s against MEASURED_PEAKS.json.
``cpu_baseline`` times the oracle port of the reference matvec
(oracle/packed_matvec.py, one core) on a bounded sample.

--impl reference times that CPU port as the reference arm (rank 0 only).
Multi-GPU (N > 1, torchrun, NCCL): the operator is sharded by subtrees
(ShardedGpuHierRep): each rank holds and streams its share and
one NCCL all-gather exchanges the multipole coefficients per matvec; the same
problem on more GPUs (strong scaling), time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

# the CPU reference leg is a single interpreter thread issuing small GEMVs
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(N=4096, d=2, kernel="log2d", n_max=64, eps=1e-8,
                 desc="cfg1: 2D N=4096 uniform [-1,1]^2, log r, leaf<=64, eps 1e-8"),
    "cfg2": dict(N=1048576, d=2, kernel="log2d", n_max=64, eps=1e-8,
                 desc="cfg2: 2D N=1048576 uniform [-1,1]^2, log r, leaf<=64, eps 1e-8"),
    "cfg3": dict(N=1048576, d=3, kernel="lap3d", n_max=64, eps=1e-6,
                 desc="cfg3: 3D N=1048576 uniform [-1,1]^3, 1/r, leaf<=64, eps 1e-6"),
    # config 5's pipeline at 1/8 of its size: jittered 128^3 grid (cfg 5: 256^3,
    # whose native build alone would take ~1.5 h of the box's 16 cores), only the
    # transfer operators stored, near + M2L evaluated on the device
    "cfg5s": dict(N=128 ** 3, d=3, kernel="lap3d", n_max=64, eps=1e-6, grid=128, store="",
                  desc="cfg5 at 1/8 size: 3D jittered 128^3 grid in [-1,1]^3, 1/r, leaf<=64, "
                       "eps 1e-6, near + M2L not stored (evaluated)"),
    # config 4's kernel and shape at 1/16 of its size (the Gaussian at eps 1e-8 is
    # near-dense: ranks ~1000 at N = 131,072, a 46 GB operator and a 36 min build)
    "cfg4s": dict(N=32768, d=3, kernel="gaussian", n_max=64, eps=1e-8,
                  desc="cfg4 at 1/16 size: 3D N=32768 uniform [-1,1]^3, Gaussian sigma 0.1 "
                       "+ 1e-6 I, leaf<=64, eps 1e-8"),
}
# BASELINE.json "metric"; config.workload names the configuration measured
METRIC = "H2* matvec/s and achieved HBM GB/s (fp64, 1/2/4/8 B200) vs ref CPU matvec"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.source = None

    def _run(self):
        # In-process NVML first: a query costs well under a millisecond, so the
        # ~0.1 s timed regions get tens of samples; nvidia-smi (tens of ms per
        # call) is the fallback.
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown,
                    pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwPowerCap]
            mx = str(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), mx] + ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.005)
            self.source = "nvml"
            return
        except Exception:
            pass
        self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def build_op(cfg, variant, n_threads=0):
    from paper_2309_14085_b200.builder import build_variant, jittered_grid, uniform_points
    if "grid" in cfg:
        pts = jittered_grid(cfg["grid"], cfg["d"], 42)
    else:
        pts = uniform_points(cfg["N"], cfg["d"], 42)
    t0 = time.perf_counter()
    op = build_variant(variant, pts, cfg["kernel"], cfg["n_max"], cfg["eps"], n_threads=n_threads,
                       store=cfg.get("store", "near,m2l"))
    return op, time.perf_counter() - t0


def cpu_port_time(op, q, budget_s=15.0, max_steps=20):
    """Oracle port of HierRep.matvec (engine.py:250-269), one core."""
    from oracle.packed_matvec import packed_matvec
    times = []
    t_start = time.perf_counter()
    while len(times) < max_steps and (time.perf_counter() - t_start) < budget_s:
        t0 = time.perf_counter()
        packed_matvec(op, q)
        times.append(time.perf_counter() - t0)
    return float(np.mean(times)), len(times)


def recompute_for(cfg, arg, op=None):
    """Which raw kernel blocks the device evaluates instead of streaming
    (csrc/h2g_p2p.cuh).  "auto": whichever the measurements say is faster
     -- log r streams (the fp64 log costs ~3.5x the bytes);
    1/r evaluates M2L (1.3x faster than streaming it) and the near field
    only for leaves of >= 48 points on average (at ~32 points streaming the
    near blocks is as fast); blocks the build did not store are always
    evaluated."""
    if cfg.get("store") == "":
        return "near,m2l"
    if arg != "auto":
        return "" if arg in ("none", "stream") else arg
    if cfg["kernel"] != "lap3d":
        return ""
    if op is not None:
        n_leaves = int(op.level_offset[op.kappa + 1] - op.level_offset[op.kappa])
        if op.N / max(1, n_leaves) >= 48:
            return "near,m2l"
    return "m2l"


def dgemm_tflops(torch, dev):
    """Measured fp64 tensor-pipe peak on this GPU (cuBLAS DGEMM 8192^3)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=f"cuda:{dev}")
    b = torch.randn(n, n, dtype=torch.float64, device=f"cuda:{dev}")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize(dev)
    del a, b
    return 2 * n ** 3 * 5 / (e0.elapsed_time(e1) * 1e-3) / 1e12


def bench_multi_rhs(rep, op, torch, dev, k=16, iters=10):
    """Batched-RHS engine (csrc/h2g_stream.cuh stream_mma_kernel, DMMA): one
    operator pass per 16 right-hand sides; fp64 TFLOP/s = 2 S k / t."""
    Q = torch.randn(op.N, k, dtype=torch.float64, device=f"cuda:{dev}")
    for _ in range(2):
        rep.matmat(Q)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        rep.matmat(Q)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / iters
    peak = dgemm_tflops(torch, dev)
    tf = 2 * op.mem_scalars * k / (ms * 1e-3) / 1e12
    return {"nrhs": k, "ms_per_block": ms, "matvec_per_s": k * 1e3 / ms,
            "fp64_tflops": tf, "dgemm_peak_tflops": peak, "tensor_frac": tf / peak,
            "hbm_roofline_tflops": 0.25 * k * _peaks()[0] / 1e3,
            "launches": rep.launches_per_matvec(k)}


def bench_gmres(rep, op, torch, dev, k=16, restart=30, max_iter=300):
    """Config 4's solve: restarted block GMRES(30) over k RHS ~ N(0,1)
    (seed 43, reference bench.py:131-136), one batched operator application
    per Arnoldi step (solver.py, CGS2), to relative residual 1e-8 or
    max_iter steps; wall-clock on the host around the device-resident solve."""
    from paper_2309_14085_b200.solver import gmres_block
    B = torch.from_numpy(np.random.default_rng(43).standard_normal((k, op.N)).T.copy()).to(
        f"cuda:{dev}")
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    X, r = gmres_block(rep.matmat, B, tol=1e-8, restart=restart, max_iter=max_iter,
                       record_residuals=False)
    torch.cuda.synchronize(dev)
    t = time.perf_counter() - t0
    R = B - rep.matmat(X)
    true_res = float((torch.linalg.vector_norm(R, dim=0) / torch.linalg.vector_norm(B, dim=0)).max())
    return {"nrhs": k, "restart": restart, "tol": 1e-8, "max_iter": max_iter, "seconds": t,
            "arnoldi_steps": r.iterations, "operator_applications": r.matvecs,
            "ms_per_step": t / max(1, r.iterations) * 1e3, "true_rel_residual_max": true_res,
            "converged": bool(true_res <= 1e-8),
            "note": "unpreconditioned GMRES(30) stagnates on exp(-r^2/0.02) + 1e-6 I; GMRES(30) "
                    "built from the reference's own solver does too (residual after 300 steps "
                    "4.6e-10 / 4.7e-4 / 3.2e-2 at N = 1024 / 2048 / 4096, "
                    "tests/golden/gmres_gauss_ref.npz)"}


def bench_variant(op, args, torch, dev, rank, world, recompute=""):
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    rep = GpuHierRep(op, device=dev, recompute=recompute)
    N = op.N
    q = np.random.default_rng(43).standard_normal(N)
    qd = torch.from_numpy(q).to(f"cuda:{dev}")
    out = torch.empty_like(qd)
    stream = torch.cuda.Stream(device=dev)
    L, plan = rep._L, rep._plan

    def step():
        L.h2g_matvec(plan, qd.data_ptr(), out.data_ptr(), N, 1, 1, stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    # per-phase CUDA-event timing on the plan stream (roofline of the GEMV kernel)
    prof = rep.profile_phases(qd, out, iters=max(3, min(args.steps, 10)))
    # e2e through the public API with pinned host buffers
    q_pin = torch.from_numpy(q).pin_memory()
    qh = q_pin.numpy()
    phi_pin = torch.empty(N, dtype=torch.float64).pin_memory().numpy()
    phi = None
    for _ in range(max(1, args.warmup // 2)):
        phi = rep.matvec(qh, out=phi_pin)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        phi = rep.matvec(qh, out=phi_pin)
    e2e_s = (time.perf_counter() - t0) / args.steps
    res = {"rep": rep, "ms": ms, "prof": prof, "clk": clk.summary(), "e2e_s": e2e_s,
           "q": q, "phi": phi, "out": out}
    if args.nrhs > 1 and not recompute:
        res["multi_rhs"] = bench_multi_rhs(rep, op, torch, dev, k=args.nrhs)
    if op.kernel.get("name") == "gaussian" and not recompute:
        res["gmres"] = bench_gmres(rep, op, torch, dev, k=max(args.nrhs, 1))
    return res


def bench_variant_sharded(op, args, torch, dev, rank, world):
    """Strong scaling: the operator split over `world` GPUs, one all-gather."""
    from paper_2309_14085_b200.sharded import ShardedGpuHierRep
    rep = ShardedGpuHierRep(op, rank, world, device=dev)
    N = op.N
    q = np.random.default_rng(43).standard_normal(N)
    qd = torch.from_numpy(q).to(f"cuda:{dev}")
    for _ in range(args.warmup):
        rep.matvec(qd)
    torch.cuda.synchronize(dev)
    torch.distributed.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize(dev)
        ev0.record()
        for _ in range(args.steps):
            rep.matvec(qd)
        ev1.record()
        torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], device=f"cuda:{dev}")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    # e2e: pinned host q -> device, sharded matvec, this rank's rows -> host
    q_pin = torch.from_numpy(q).pin_memory()
    phi_pin = torch.empty(N, dtype=torch.float64).pin_memory()
    torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        qd2 = q_pin.to(f"cuda:{dev}", non_blocking=True)
        phi_pin.copy_(rep.matvec(qd2), non_blocking=True)
        torch.cuda.synchronize(dev)
    e2e = torch.tensor([(time.perf_counter() - t0) / args.steps], device=f"cuda:{dev}")
    torch.distributed.all_reduce(e2e, op=torch.distributed.ReduceOp.MAX)
    torch.distributed.barrier()
    return {"rep": rep, "ms": ms, "prof": [], "clk": clk.summary(), "e2e_s": float(e2e.item()),
            "q": q, "shard": rep.info}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--variants", default="h2star-bt,h2plusH-star")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--recompute", default="auto",
                    help="raw kernel blocks evaluated on the device: auto|none|near|m2l|near,m2l")
    ap.add_argument("--nrhs", type=int, default=16,
                    help="also time the batched-RHS engine with this many right-hand sides")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = CONFIGS[args.config]
    variants = [v for v in args.variants.split(",") if v]
    rank, world, local = dist_env()
    n_threads = max(1, (os.cpu_count() or 1) // max(1, world))

    if args.impl == "reference":
        if rank != 0:
            return
        op, tb = build_op(cfg, variants[0], n_threads=os.cpu_count() or 1)
        q = np.random.default_rng(43).standard_normal(cfg["N"])
        from oracle.packed_matvec import packed_matvec
        for _ in range(min(args.warmup, 1)):
            packed_matvec(op, q)
        budget = 240.0
        times = []
        t_all = time.perf_counter()
        for _ in range(args.steps):
            t0 = time.perf_counter()
            packed_matvec(op, q)
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - t_all > budget:
                break
        s = float(np.mean(times))
        v = 1.0 / s
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "matvec/s",
                "n_gpus": args.gpus, "steps": len(times), "warmup": min(args.warmup, 1),
                "ms_per_step": s * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": cfg["desc"], "variant": variants[0], "N": cfg["N"],
                           "mem_scalars": int(op.mem_scalars),
                           "operator": "native build (libh2b.so), identical structure/ranks "
                                       "to the reference build"},
                "cpu_baseline": {"value": v, "unit": "matvec/s", "cores": 1, "kind": "port",
                                 "sample": f"{len(times)} full matvecs of the oracle port "
                                           "(oracle/packed_matvec.py: reference loop structure, "
                                           "numpy @ per block, OPENBLAS_NUM_THREADS=1)"},
                "e2e": {"value": v, "unit": "matvec/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    if world > 1:
        torch.distributed.init_process_group("nccl")
    dev = local if torch.cuda.device_count() > local else 0
    torch.cuda.set_device(dev)

    results = {}
    for v in variants:
        op, tb = build_op(cfg, v, n_threads=n_threads)
        if world > 1:
            r = bench_variant_sharded(op, args, torch, dev, rank, world)
        else:
            r = bench_variant(op, args, torch, dev, rank, world,
                              recompute=recompute_for(cfg, args.recompute, op))
        r["op"] = op
        r["build_s"] = tb
        results[v] = r
        if v != variants[0]:
            r["rep"].close()

    head = variants[0]
    R = results[head]
    op, rep = R["op"], R["rep"]
    alg_bytes = 8 * op.mem_scalars + 16 * op.N
    value = 1e3 / R["ms"]  # whole-job matvecs/s (one operator, sharded over `world` GPUs)
    peak, peak_src = _peaks()
    if world == 1:
        # roofline: streaming GEMV kernel phases (algorithmic bytes / event time)
        gemv = [p for p in R["prof"] if p["phase"] not in ("gather", "scatter", "blr_reduce")]
        rc = recompute_for(cfg, args.recompute, op)
        k_bytes = sum(p["bytes"] for p in gemv)
        k_ms_serial = sum(p["ms"] for p in gemv)
        # the GEMV launches overlap at phase boundaries (programmatic dependent
        # launch), so their average duration is their span inside the timed
        # step: step time minus the gather / scatter kernels (event-timed)
        edge_ms = sum(p["ms"] for p in R["prof"] if p["phase"] in ("gather", "scatter"))
        k_ms = max(R["ms"] - edge_ms, 1e-9)
        achieved = k_bytes / (k_ms * 1e-3) / 1e9
        achieved_serial = k_bytes / (k_ms_serial * 1e-3) / 1e9
        dom = max(gemv, key=lambda p: p["ms"])
        dom = {"name": dom["phase"], "ms": dom["ms"],
               "GBps": dom["bytes"] / (dom["ms"] * 1e-3) / 1e9}
        kernel = ("stream_gemv_kernel (all GEMV phases)" if not rc else
                  f"stream_gemv_kernel + p2p_tasks_kernel (all phases; {rc} blocks evaluated "
                  "on the fp64 pipe: achieved = stored-representation bytes / time, may "
                  "exceed the HBM peak)")
    else:
        # per-GPU share of the algorithmic bytes over the whole (max-over-ranks) step
        achieved = alg_bytes / world / (R["ms"] * 1e-3) / 1e9
        achieved_serial = None
        dom = None
        kernel = "whole sharded matvec per GPU (all phases + NCCL all-gather)"
    traffic = None
    rc_used = recompute_for(cfg, args.recompute, op) if world == 1 else ""
    tpath = os.path.join(ROOT, "profiles",
                         f"traffic_{args.config}_{head}{'_eval' if rc_used else ''}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": R["ms"],
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (uniform_points seed 42, q ~ N(0,1) seed 43)",
        "config": {"workload": cfg["desc"], "variant": head, "N": op.N, "kappa": op.kappa,
                   "mem_scalars": int(op.mem_scalars), "alg_bytes": alg_bytes,
                   "parallelism": f"subtree-sharded x{world}" if world > 1 else "single",
                   "l2": "operator > L2 (no flush)", "build_s": round(R["build_s"], 2),
                   "evaluated_blocks": recompute_for(cfg, args.recompute, op) or "none"},
        "achieved_GBps": alg_bytes / (R["ms"] * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "launches_per_step": (rep.launches_per_matvec() - 2) if world == 1 else None,
                     "achieved_phase_by_phase": achieved_serial if world == 1 else None,
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": kernel, "dominant_phase": dom},
        "e2e": {"value": 1.0 / R["e2e_s"], "unit": "matvec/s",
                "h2d_bytes_per_step": 8 * op.N, "d2h_bytes_per_step": 8 * op.N},
        "gpu_launches": args.steps * rep.launches_per_matvec(),
        "clocks": R["clk"],
        "phases_us": {p["phase"]: round(p["ms"] * 1e3, 1) for p in R["prof"]},
    }
    if world > 1:
        line["shard"] = R["shard"]
    if "multi_rhs" in R:
        line["multi_rhs"] = R["multi_rhs"]
    if "gmres" in R:
        line["gmres"] = R["gmres"]
    others = {}
    for v in variants[1:]:
        r = results[v]
        others[v] = {"ms_per_step": r["ms"], "matvec_per_s": 1e3 / r["ms"],
                     "mem_scalars": int(r["op"].mem_scalars),
                     "achieved_GBps": (8 * r["op"].mem_scalars + 16 * r["op"].N) / (r["ms"] * 1e-3) / 1e9,
                     "e2e_matvec_per_s": 1.0 / r["e2e_s"], "build_s": round(r["build_s"], 2)}
    if others:
        line["variants"] = others
    if rank == 0 and world == 1 and cfg.get("store") == "":
        line["cpu_baseline"] = {"value": None, "unit": "matvec/s", "cores": 1, "kind": "port",
                                "sample": "not run: the operator's near/M2L blocks are not stored "
                                          "and the numpy oracle would evaluate ~10^10 entries"}
    elif rank == 0 and world == 1:
        t_cpu, n_cpu = cpu_port_time(op, R["q"], budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": 1.0 / t_cpu, "unit": "matvec/s", "cores": 1, "kind": "port",
                                "sample": f"{n_cpu} full matvecs of the oracle port on the same "
                                          "operator (oracle/packed_matvec.py, 1 BLAS thread)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    rep.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
