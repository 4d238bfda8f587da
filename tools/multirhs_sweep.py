"""Multi-RHS (batched fp64 tensor-pipe) engine timing + block GMRES on a
Gaussian (cfg-4 shaped) operator.  Diagnostics; bench.py is the contract.

    python tools/multirhs_sweep.py [N_gauss]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def dgemm_peak(torch):
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    return 2 * n ** 3 * 5 / (e0.elapsed_time(e1) * 1e-3) / 1e12


def time_matmat(torch, rep, N, k, it=10):
    Q = torch.randn(N, k, dtype=torch.float64, device="cuda")
    for _ in range(2):
        rep.matmat(Q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        rep.matmat(Q)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


def main():
    import torch
    from paper_2309_14085_b200.builder import build_variant, uniform_points
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    from paper_2309_14085_b200.solver import gmres_block
    peak = dgemm_peak(torch)
    print(json.dumps({"dgemm_tflops": peak}), flush=True)
    for (N, d, ker, eps) in ((1048576, 2, "log2d", 1e-8), (262144, 3, "lap3d", 1e-6)):
        op = build_variant("h2star-bt", uniform_points(N, d, 42), ker, 64, eps)
        with GpuHierRep(op) as rep:
            S = op.mem_scalars
            out = {"N": N, "kernel": ker}
            for k in (1, 8, 16):
                ms = time_matmat(torch, rep, N, k)
                out[f"k{k}_ms"] = ms
                out[f"k{k}_tflops"] = 2 * S * k / (ms * 1e-3) / 1e12
                out[f"k{k}_per_rhs_ms"] = ms / k
            out["tensor_frac_k16"] = out["k16_tflops"] / peak
            print(json.dumps(out), flush=True)
    Ng = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    t0 = time.time()
    op = build_variant("h2star-bt", uniform_points(Ng, 3, 42), "gaussian", 64, 1e-8)
    tb = time.time() - t0
    with GpuHierRep(op) as rep:
        B = torch.from_numpy(np.random.default_rng(43).standard_normal((16, Ng)).T.copy()).cuda()
        ms16 = time_matmat(torch, rep, Ng, 16)
        torch.cuda.synchronize()
        t0 = time.time()
        X, r = gmres_block(rep.matmat, B, tol=1e-8, restart=30, max_iter=600,
                           record_residuals=False)
        torch.cuda.synchronize()
        tg = time.time() - t0
        R = B - rep.matmat(X)
        true_res = (torch.linalg.vector_norm(R, dim=0) / torch.linalg.vector_norm(B, dim=0)).max()
    print(json.dumps({"gauss_N": Ng, "build_s": tb, "mem_GB": op.mem_scalars * 8e-9,
                      "k16_ms": ms16, "k16_tflops": 2 * op.mem_scalars * 16 / (ms16 * 1e-3) / 1e12,
                      "gmres_s": tg, "iterations": r.iterations, "matvecs": r.matvecs,
                      "restarts": r.restarts, "residual_est": r.residual,
                      "true_residual": float(true_res), "converged": r.converged,
                      "ms_per_step": tg / max(1, r.iterations) * 1e3}), flush=True)


if __name__ == "__main__":
    main()
