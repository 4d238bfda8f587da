"""Hybrid M2L phases on one B200: a share of each evaluated level's targets
streamed on the streaming engine while the P2P engine evaluates the rest,
concurrently (h2g_plan.cu, Phase.hybrid; env H2G_M2L_STREAM_SHARE).

    python tools/hybrid_sweep.py [cfg3|N,d,kernel,eps] [modes...]

modes: "hF" = hybrid phases with share F of the M2L entries streamed on the
streaming engine beside the P2P engine; "sF" = m2l_recompute_share F (share
EVALUATED; the rest of every target's M2L blocks TMA-staged inside the P2P
tasks); "s1" = all evaluated.  Prints one JSON line per mode: ms per matvec (CUDA events, 20 matvecs after
5 warm-ups), per-phase us, error vs the all-streamed result.  Diagnostics
only; bench.py is the measured contract.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2309_14085_b200.builder import build_variant, uniform_points
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    spec = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    presets = {"cfg3": (1048576, 3, "lap3d", 1e-6)}
    if spec in presets:
        N, d, kernel, eps = presets[spec]
    else:
        a = spec.split(",")
        N, d, kernel, eps = int(a[0]), int(a[1]), a[2], float(a[3])
    modes = sys.argv[2:] or ["s1", "s0.7", "s0.6", "s0.5"]
    t0 = time.time()
    op = build_variant("h2star-bt", uniform_points(N, d, 42), kernel, 64, eps)
    print(json.dumps({"build_s": time.time() - t0, "N": N, "mem_GB": op.mem_scalars * 8e-9}),
          flush=True)
    q = np.random.default_rng(43).standard_normal(N)
    qd = torch.from_numpy(q).cuda()
    out = torch.empty_like(qd)
    with GpuHierRep(op) as rep:
        base = rep.matvec(q)
    stream = torch.cuda.Stream()
    for mode in modes:
        sh = float(mode[1:])
        if mode[0] == "h":
            os.environ["H2G_M2L_STREAM_SHARE"] = str(sh)
            kw = {}
        else:
            os.environ.pop("H2G_M2L_STREAM_SHARE", None)
            kw = {"m2l_share": sh}
        with GpuHierRep(op, recompute="m2l", **kw) as rep:
            L, plan = rep._L, rep._plan
            for _ in range(5):
                L.h2g_matvec(plan, qd.data_ptr(), out.data_ptr(), N, 1, 1, stream.cuda_stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(20):
                L.h2g_matvec(plan, qd.data_ptr(), out.data_ptr(), N, 1, 1, stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            phi = out.cpu().numpy().copy()
            prof = rep.profile_phases(qd, out, iters=5)
            err = float(np.linalg.norm(phi - base) / np.linalg.norm(base))
            print(json.dumps({"mode": mode, "ms": ms, "matvec_per_s": 1e3 / ms, "err_vs_streamed": err,
                              "launches": rep.launches_per_matvec(),
                              "phases_us": {p["phase"]: round(p["ms"] * 1e3, 1) for p in prof}}),
                  flush=True)
    os.environ.pop("H2G_M2L_STREAM_SHARE", None)


if __name__ == "__main__":
    main()
