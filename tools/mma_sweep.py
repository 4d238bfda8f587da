"""Sweep of diagnostic libh2g variants (tools/build_variant.sh) over the
batched-RHS (DMMA) engine: the operator is built once, exported to a scratch
directory and loaded (mmap) by one subprocess per variant, which prints the
per-phase times of a 16-RHS pass and the timed matmat.  Diagnostics.

    python tools/mma_sweep.py N dim variant [variant ...]      ("base" = the in-tree library)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(path, N):
    import torch
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    from paper_2309_14085_b200.packed import PackedOperator
    op = PackedOperator.load_dir(path)
    with GpuHierRep(op) as rep:
        Q = torch.randn(N, 16, dtype=torch.float64, device="cuda")
        for _ in range(3):
            rep.matmat(Q)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            rep.matmat(Q)
        e1.record()
        torch.cuda.synchronize()
        out = {"variant": os.environ.get("SWEEP_VARIANT", "base"),
               "matmat16_ms": e0.elapsed_time(e1) / 10,
               "hbm_floor_ms": 8 * op.mem_scalars / 6.545e12 * 1e3}
        ph = rep.profile_phases_batched(16, iters=10)
        out["phases_ms"] = {r["phase"]: round(r["ms"], 4) for r in ph}
        out["phases_GBps"] = {r["phase"]: round(r["bytes"] / (r["ms"] * 1e-3) / 1e9, 0)
                              for r in ph if r["ms"] > 0.02}
        out["sum_phases_ms"] = sum(r["ms"] for r in ph)
    print(json.dumps(out), flush=True)


def main():
    N, d = int(sys.argv[1]), int(sys.argv[2])
    variants = sys.argv[3:] or ["base"]
    from paper_2309_14085_b200.builder import build_variant, uniform_points
    kern, eps = ("log2d", 1e-8) if d == 2 else ("lap3d", 1e-6)
    op = build_variant("h2star-bt", uniform_points(N, d, 42), kern, 64, eps)
    path = f"/tmp/mma_sweep_{N}_{d}"
    op.save_dir(path)
    del op
    for v in variants:
        env = dict(os.environ)
        lib, _, envs = v.partition(":")          # "lib:ENV=VAL,ENV=VAL"
        for kv in filter(None, envs.split(",")):
            k, _, val = kv.partition("=")
            env[k] = val
        env["SWEEP_VARIANT"] = v
        if lib != "base":
            env["H2G_LIB_PATH"] = os.path.join(ROOT, "paper_2309_14085_b200", "lib", "var",
                                               f"libh2g_{lib}.so")
        subprocess.run([sys.executable, __file__, "--child", path, str(N)], env=env, timeout=600)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]))
    else:
        main()
