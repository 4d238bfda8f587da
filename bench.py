"""Benchmark: H2* matvec on B200 (BASELINE.json configs[2], the north-star
HBM-roofline config).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg3] [--variants h2star-bt] [--recompute auto]

Workload (configs[2]): 3D, N = 1,048,576 points i.i.d. uniform in [-1,1]^3
(seed 42, reference bench.py:41), K(x,y) = 1/|x-y| (InverseR,
kernels.py:74-81), octree leaf <= 64, NCA tolerance 1e-6, H2*(b+t), single
RHS q ~ N(0,1) (seed 43).  The operator (89.8 GB, every block stored) is
built on the box by the native builder (libh2b.so), which restates the
reference construction (identical trees, ranks and pivots on every golden
fixture); the reference's own Python build is infeasible at this size.

A step is one matvec phi = K~ q.  ``value`` = matvecs/s of the headline
variant in the evaluation mode ``--recompute auto`` picks (cfg 3: the M2L
blocks K[t_i, s_o] evaluated on the fp64 pipe, everything else streamed),
device-timed with CUDA events on the plan's stream, inputs resident in HBM;
the operator is far larger than L2 (126 MB), so no flush is needed.  ``e2e``
is the same metric through the public API (GpuHierRep.matvec(q, out=phi) on
pinned host vectors: H2D copy, matvec, D2H copy inside the timed region);
``e2e.reference_call_shape`` is GpuHierRep.matvec(q) on a pageable numpy q
returning a fresh phi (the reference's own call shape).  ``roofline``:
achieved = (8 S + 16 N) / step time (SURVEY §8(d), S = rep.mem_scalars)
against MEASURED_PEAKS.json; with evaluated blocks that rate is
"stored-equivalent" and the DRAM traffic / fp64-pipe figures say what bounds
the step.  ``variants.streamed`` is the same operator with every block read
from HBM (the pure HBM fraction).  ``cpu_baseline`` times the oracle port of
the reference matvec (oracle/cpu_reference.py, one core) on a bounded
sample (full upward pass + one 1/64 subtree's downward pass, extrapolated).

--impl reference times that CPU port as the reference arm (rank 0 only) on
an operator exported by a separate build process (no repo .so in the timing
process).  Multi-GPU (N > 1, torchrun, NCCL): the operator is sharded by
subtrees (ShardedGpuHierRep) with the same evaluation policy;
one NCCL all-gather exchanges the multipole coefficients per matvec; the
same problem on more GPUs (strong scaling), time = max over ranks.
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


DEFAULT_VARIANTS = {"cfg1": "h2star-bt,h2plusH-star", "cfg2": "h2star-bt,h2plusH-star",
                    "cfg3": "h2star-bt", "cfg4s": "h2star-bt", "cfg5s": "h2star-bt"}


def build_op(cfg, variant, n_threads=0, store=None):
    from paper_2309_14085_b200.builder import build_variant, jittered_grid, uniform_points
    if "grid" in cfg:
        pts = jittered_grid(cfg["grid"], cfg["d"], 42)
    else:
        pts = uniform_points(cfg["N"], cfg["d"], 42)
    t0 = time.perf_counter()
    op = build_variant(variant, pts, cfg["kernel"], cfg["n_max"], cfg["eps"], n_threads=n_threads,
                       store=cfg.get("store", "near,m2l") if store is None else store)
    return op, time.perf_counter() - t0


def build_op_shared(cfg, variant, rank, world, barrier, tmp_root="/tmp"):
    """N > 1: ONE native build for the node instead of one per rank.  Rank 0
    runs the NCA pivot search with every host thread and exports the operator
    without its raw kernel blocks (store="": transfer operators, pivots,
    points; ~1 GB); after the barrier every rank loads the export.  Configs
    that store their blocks re-evaluate them natively (builder.
    materialize_blocks: bitwise the blocks of a stored build, seconds) -- the
    caller does that one rank at a time so the node never holds more than one
    full operator in host memory beside the plans' uploads."""
    import shutil
    from paper_2309_14085_b200.packed import PackedOperator
    path = os.path.join(tmp_root, f"h2g_bench_{cfg['N']}_{cfg['kernel']}_{variant}")
    tb = 0.0
    if rank == 0:
        shutil.rmtree(path, ignore_errors=True)
        op0, tb = build_op(cfg, variant, n_threads=os.cpu_count() or 1, store="")
        op0.save_dir(path)
        del op0
    barrier()
    return PackedOperator.load_dir(path), tb


def config_dict(cfg, variant, N, kappa, mem_scalars, world):
    """The workload (identical in both arms)."""
    return {"workload": cfg["desc"], "variant": variant, "N": int(N), "kappa": int(kappa),
            "mem_scalars": int(mem_scalars), "alg_bytes": int(8 * mem_scalars + 16 * N),
            "parallelism": f"subtree-sharded x{world}" if world > 1 else "single",
            "l2": "operator > L2 (no flush)"}


def export_for_reference(cfg_name, variant, path, n_threads):
    """Separate build process: the native builder writes the operator's
    transfer operators, pivots and points (store="": no raw kernel block) to
    ``path``; the reference arm then loads it without mapping any repo .so."""
    code = ("import sys, json, time; sys.path.insert(0, %r); import bench; "
            "cfg = bench.CONFIGS[%r]; op, tb = bench.build_op(cfg, %r, %d, store=''); "
            "op.save(%r); print(json.dumps({'build_s': tb}))"
            % (ROOT, cfg_name, variant, n_threads, path))
    out = subprocess.run([sys.executable, "-c", code], check=True, capture_output=True, text=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_port_time(op, q, budget_s=15.0, max_steps=20):
    """Oracle port of HierRep.matvec (engine.py:250-269), one core, on the
    bounded sample of oracle/cpu_reference.py."""
    from oracle.cpu_reference import time_sampled_matvec
    return time_sampled_matvec(op, q, steps=max_steps, warmup=0, budget_s=budget_s)


# Share of the STORED M2L entries the P2P engine evaluates when it evaluates
# M2L; the rest of every target's blocks stream (TMA-staged, multiplied by the
# P2P CTAs' streaming warps) inside the same tasks, so HBM and the fp64 pipe
# work at once (tools/variant_sweep.py, cfg 3: 1.0 -> 11.44 ms, 0.7 -> 10.07,
# 0.6 -> 10.04, 0.5 -> 10.34).
M2L_EVAL_SHARE = 0.6


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


def _time_steps(step, args, torch, dev, stream, world):
    """W warm-ups, then K steps between CUDA events on ``stream`` (clocks
    sampled throughout), max over ranks."""
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
    return ms, clk.summary()


def bench_variant(op, args, torch, dev, rank, world, recompute="", e2e=True):
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    rep = GpuHierRep(op, device=dev, recompute=recompute, m2l_share=args.m2l_share)
    N = op.N
    q = np.random.default_rng(43).standard_normal(N)
    qd = torch.from_numpy(q).to(f"cuda:{dev}")
    out = torch.empty_like(qd)
    stream = torch.cuda.Stream(device=dev)
    L, plan = rep._L, rep._plan

    def step():
        L.h2g_matvec(plan, qd.data_ptr(), out.data_ptr(), N, 1, 1, stream.cuda_stream)

    ms, clk = _time_steps(step, args, torch, dev, stream, world)
    # per-phase CUDA-event timing on the plan stream (which phase dominates)
    prof = rep.profile_phases(qd, out, iters=max(3, min(args.steps, 10)))
    res = {"rep": rep, "ms": ms, "prof": prof, "clk": clk, "q": q, "out": out}
    if args.nrhs > 1:
        res["multi_rhs"] = bench_multi_rhs(rep, op, torch, dev, k=args.nrhs)
        if recompute:
            res["multi_rhs"]["engine"] = ("stored blocks on the DMMA engine, evaluated blocks on "
                                          "the batched P2P engine (one evaluation per entry for "
                                          "all right-hand sides)")
    if not e2e:
        return res
    # e2e through the public API with pinned host buffers (out=)
    q_pin = torch.from_numpy(q).pin_memory()
    qh = q_pin.numpy()
    phi_pin = torch.empty(N, dtype=torch.float64).pin_memory().numpy()
    for _ in range(max(1, args.warmup // 2)):
        rep.matvec(qh, out=phi_pin)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rep.matvec(qh, out=phi_pin)
    res["e2e_s"] = (time.perf_counter() - t0) / args.steps
    # the reference's call shape: pageable numpy q, freshly allocated phi
    qp = np.array(q)
    rep.matvec(qp)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rep.matvec(qp)
    res["e2e_ref_shape_s"] = (time.perf_counter() - t0) / args.steps
    if op.kernel.get("name") == "gaussian" and not recompute:
        res["gmres"] = bench_gmres(rep, op, torch, dev, k=max(args.nrhs, 1))
    return res


def bench_setup_sharded(op, args, dev, rank, world, recompute=""):
    """This rank's sharded plan (uploads only the blocks its tasks read)."""
    from paper_2309_14085_b200.sharded import ShardedGpuHierRep
    return ShardedGpuHierRep(op, rank, world, device=dev, recompute=recompute,
                             m2l_share=args.m2l_share)


def bench_variant_sharded(rep, op, args, torch, dev, rank, world):
    """Strong scaling: the operator split over `world` GPUs, one all-gather
    overlapped with the owned near field."""
    N = op.N
    q = np.random.default_rng(43).standard_normal(N)
    qd = torch.from_numpy(q).to(f"cuda:{dev}")
    stream = torch.cuda.current_stream(dev)
    ms, clk = _time_steps(lambda: rep.matvec(qd), args, torch, dev, stream, world)
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
    return {"rep": rep, "ms": ms, "prof": [], "clk": clk, "e2e_s": float(e2e.item()),
            "q": q, "shard": rep.info}


def _profile_json(name):
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as fh:
            return json.load(fh), os.path.relpath(path, ROOT)
    except Exception:
        return None, None


def reference_arm(args, cfg, variants, world):
    """--impl reference: the oracle port of the reference matvec on the box's
    host (rank 0), on an operator a SEPARATE build process exported (so this
    process never maps a repo .so), same config / warmup as our arm."""
    import tempfile
    n_threads = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "op.npz")
        info = export_for_reference(args.config, variants[0], path, n_threads)
        from paper_2309_14085_b200.packed import PackedOperator
        op = PackedOperator.load(path)
    q = np.random.default_rng(43).standard_normal(cfg["N"])
    from oracle.cpu_reference import time_sampled_matvec
    r = time_sampled_matvec(op, q, steps=args.steps, warmup=args.warmup, budget_s=args.ref_budget)
    v = r["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "matvec/s",
            "n_gpus": world, "steps": r["steps"], "warmup": args.warmup,
            "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (uniform_points seed 42, q ~ N(0,1) seed 43)",
            "config": config_dict(cfg, variants[0], op.N, op.kappa, op.mem_scalars, world),
            "operator_source": ("native build in a separate process (libh2b.so), exported with "
                                "store='' (transfer operators + NCA pivots + points; identical "
                                "trees, ranks and pivots to the reference build); this process "
                                f"maps no repo .so; export build {info['build_s']:.1f} s"),
            "cpu_baseline": {"value": v, "unit": "matvec/s", "cores": 1, "kind": "port",
                             "sample": r["sample"]},
            "e2e": {"value": v, "unit": "matvec/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "timing": {k: r[k] for k in ("t_up_s", "t_down_sample_s", "sampled_leaves", "leaves")}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--variants", default=None, help="default: per config (cfg3: h2star-bt)")
    ap.add_argument("--cpu-budget", type=float, default=60.0)
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="--impl reference: stop timing after this many seconds")
    ap.add_argument("--recompute", default="auto",
                    help="raw kernel blocks evaluated on the device: auto|none|near|m2l|near,m2l")
    ap.add_argument("--streamed-variant", type=int, default=1,
                    help="also time the all-streamed plan (pure HBM fraction) when the headline "
                         "evaluates blocks")
    ap.add_argument("--m2l-share", type=float, default=M2L_EVAL_SHARE,
                    help="share of the stored M2L entries evaluated when M2L is evaluated "
                         "(the rest streams inside the same P2P tasks); 1 = all evaluated")
    ap.add_argument("--nrhs", type=int, default=16,
                    help="also time the batched-RHS engine with this many right-hand sides")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = CONFIGS[args.config]
    variants = [v for v in (args.variants or DEFAULT_VARIANTS[args.config]).split(",") if v]
    rank, world, local = dist_env()
    n_threads = max(1, (os.cpu_count() or 1) // max(1, world))

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, cfg, variants, world)
        return

    import torch
    if world > 1:
        import datetime
        # rank 0 builds the operator for the node while the others wait
        torch.distributed.init_process_group("nccl", timeout=datetime.timedelta(hours=2))
    dev = local if torch.cuda.device_count() > local else 0
    torch.cuda.set_device(dev)

    results = {}
    for v in variants:
        if world > 1:
            from paper_2309_14085_b200.builder import materialize_blocks
            op, tb = build_op_shared(cfg, v, rank, world, torch.distributed.barrier)
            rc = recompute_for(cfg, args.recompute, op)
            r = None
            for turn in range(world):  # one full operator in host memory at a time
                if turn == rank:
                    full = op if cfg.get("store") == "" else materialize_blocks(op)
                    r = bench_setup_sharded(full, args, dev, rank, world, recompute=rc)
                    del full
                torch.distributed.barrier()
            r = bench_variant_sharded(r, op, args, torch, dev, rank, world)
        else:
            op, tb = build_op(cfg, v, n_threads=n_threads)
            rc = recompute_for(cfg, args.recompute, op)
            r = bench_variant(op, args, torch, dev, rank, world, recompute=rc)
        r["op"], r["build_s"], r["rc"] = op, tb, rc
        if v == variants[0] and rc and world == 1 and args.streamed_variant and cfg.get("store") != "":
            # the same operator with every block read from HBM: the pure HBM roofline
            s = bench_variant(op, args, torch, dev, rank, world, recompute="", e2e=False)
            s["rep"].close()
            r["streamed"] = s
        results[v] = r
        if v != variants[0]:
            r["rep"].close()

    head = variants[0]
    R = results[head]
    op, rep, rc = R["op"], R["rep"], R["rc"]
    S, N = int(op.mem_scalars), int(op.N)
    alg_bytes = 8 * S + 16 * N
    value = 1e3 / R["ms"]  # whole-job matvecs/s (one operator, sharded over `world` GPUs)
    peak, peak_src = _peaks()

    def span_ms(r):  # the GEMV/P2P launches between the gather and scatter kernels
        edge = sum(p["ms"] for p in r["prof"] if p["phase"] in ("gather", "scatter"))
        return max(r["ms"] - edge, 1e-9)

    achieved = alg_bytes / world / (R["ms"] * 1e-3) / 1e9  # per GPU
    roof = {"bound": "fp64+hbm" if rc else "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
            "achieved_basis": "(8 S + 16 N) / step time, S = rep.mem_scalars (SURVEY §8(d))"
                              + (" per GPU" if world > 1 else "")}
    if world == 1:
        roof["kernel_span_achieved"] = 8 * S / (span_ms(R) * 1e-3) / 1e9
        roof["kernel_span_frac"] = roof["kernel_span_achieved"] / peak
        roof["launches_per_step"] = rep.launches_per_matvec() - 2
        p2p_ms = sum(p["ms"] for p in R["prof"] if _is_p2p_phase(p["phase"], rc))
        tot_ms = sum(p["ms"] for p in R["prof"]) or 1.0
        dom = max((p for p in R["prof"] if p["phase"] not in ("gather", "scatter")),
                  key=lambda p: p["ms"])
        roof["dominant_phase"] = {"name": dom["phase"], "ms": dom["ms"],
                                  "engine": "p2p_tasks_kernel" if _is_p2p_phase(dom["phase"], rc)
                                  else "stream_gemv_kernel"}
        roof["kernel_share"] = {"p2p_tasks_kernel": p2p_ms / tot_ms,
                                "stream_gemv_kernel": 1.0 - p2p_ms / tot_ms}
        if rc:
            roof["note"] = (f"{rc} blocks are evaluated on the fp64 pipe, never read: achieved is "
                            "the stored-equivalent rate and may exceed the HBM peak; dram_frac "
                            "(ncu DRAM bytes of the timed build / step time / peak) is the HBM "
                            "utilisation and fp64_pipe_frac the P2P kernel's fp64-pipe "
                            "utilisation (ncu)")
    tname = f"traffic_{args.config}_{head}{'_eval' if rc else ''}.json"
    tj, tsrc = _profile_json(tname)
    roof["traffic"] = tj.get("dram_bytes_per_launch") if tj else None
    if tj and world == 1:
        roof["traffic_source"] = tsrc
        roof["dram_frac"] = roof["traffic"] / (R["ms"] * 1e-3) / 1e9 / peak
    pj, psrc = _profile_json(f"p2p_{args.config}_{head}.json")
    if rc and pj and world == 1:
        roof["fp64_pipe_frac"] = pj.get("fp64_pipe_frac")
        roof["fp64_source"] = psrc
    line = {
        "metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": R["ms"],
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (uniform_points seed 42, q ~ N(0,1) seed 43)",
        "config": config_dict(cfg, head, N, op.kappa, S, world),
        "evaluated_blocks": rc or "none",
        "m2l_eval_share": args.m2l_share if "m2l" in (rc or "") and cfg.get("store") != "" else None,
        "build_s": round(R["build_s"], 2),
        "achieved_GBps": alg_bytes / (R["ms"] * 1e-3) / 1e9,
        "roofline": roof,
        "e2e": {"value": 1.0 / R["e2e_s"], "unit": "matvec/s",
                "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N},
        "gpu_launches": args.steps * rep.launches_per_matvec(),
        "clocks": R["clk"],
        "phases_us": {p["phase"]: round(p["ms"] * 1e3, 1) for p in R["prof"]},
    }
    if "e2e_ref_shape_s" in R:
        line["e2e"]["reference_call_shape"] = {
            "value": 1.0 / R["e2e_ref_shape_s"], "unit": "matvec/s",
            "call": "GpuHierRep.matvec(q) on a pageable numpy q, fresh phi (engine.py:250-269)"}
        line["e2e"]["call"] = "GpuHierRep.matvec(q, out=phi) on pinned host buffers"
    if world > 1:
        line["shard"] = R["shard"]
    for key in ("multi_rhs", "gmres"):
        if key in R:
            line[key] = R[key]
    others = {}
    if "streamed" in R:
        st = R["streamed"]
        others["streamed"] = {
            "evaluated_blocks": "none", "ms_per_step": st["ms"], "matvec_per_s": 1e3 / st["ms"],
            "hbm_achieved_GBps": alg_bytes / (st["ms"] * 1e-3) / 1e9,
            "hbm_frac": alg_bytes / (st["ms"] * 1e-3) / 1e9 / peak,
            "kernel_span_frac": 8 * S / (span_ms(st) * 1e-3) / 1e9 / peak,
            "clocks": st["clk"],
            "phases_us": {p["phase"]: round(p["ms"] * 1e3, 1) for p in st["prof"]}}
        tj2, tsrc2 = _profile_json(f"traffic_{args.config}_{head}.json")
        if tj2:
            others["streamed"]["traffic"] = tj2.get("dram_bytes_per_launch")
        if "multi_rhs" in st:
            others["streamed"]["multi_rhs"] = st["multi_rhs"]
    for v in variants[1:]:
        r = results[v]
        b = 8 * r["op"].mem_scalars + 16 * r["op"].N
        others[v] = {"ms_per_step": r["ms"], "matvec_per_s": 1e3 / r["ms"],
                     "mem_scalars": int(r["op"].mem_scalars), "evaluated_blocks": r["rc"] or "none",
                     "achieved_GBps": b / (r["ms"] * 1e-3) / 1e9, "frac": b / (r["ms"] * 1e-3) / 1e9 / peak,
                     "e2e_matvec_per_s": 1.0 / r["e2e_s"], "build_s": round(r["build_s"], 2)}
    if others:
        line["variants"] = others
    if rank == 0 and world == 1:
        t = cpu_port_time(op, R["q"], budget_s=args.cpu_budget, max_steps=1)
        line["cpu_baseline"] = {"value": t["value"], "unit": "matvec/s", "cores": 1, "kind": "port",
                                "sample": t["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    rep.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def _is_p2p_phase(name, rc):
    """Phases the P2P (kernel-evaluation) engine runs under the recompute policy."""
    if name.endswith("_red"):
        return False
    return ("m2l" in (rc or "") and name.startswith("down_l")) or (
        "near" in (rc or "") and name == "leaf")


if __name__ == "__main__":
    main()
