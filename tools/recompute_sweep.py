"""Per-phase timing of the streamed vs evaluated (P2P) engines on one B200.

    python tools/recompute_sweep.py [cfg3|cfg2|N,d,kernel,eps] [modes...]

modes: "stream", "near", "m2l", "near,m2l", "near,m2l@0.6" (hybrid share).
Prints one JSON line per mode (ms per matvec, per-phase us, error vs the
streamed result).  Diagnostics only; bench.py is the measured contract.
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
    presets = {"cfg3": (1048576, 3, "lap3d", 1e-6), "cfg2": (1048576, 2, "log2d", 1e-8)}
    if spec in presets:
        N, d, kernel, eps = presets[spec]
    else:
        a = spec.split(",")
        N, d, kernel, eps = int(a[0]), int(a[1]), a[2], float(a[3])
    modes = sys.argv[2:] or ["stream", "near", "m2l", "near,m2l", "near,m2l@0.6"]
    t0 = time.time()
    op = build_variant("h2star-bt", uniform_points(N, d, 42), kernel, 64, eps)
    print(json.dumps({"build_s": time.time() - t0, "N": N, "mem_GB": op.mem_scalars * 8e-9}),
          flush=True)
    q = np.random.default_rng(43).standard_normal(N)
    qd = torch.from_numpy(q).cuda()
    out = torch.empty_like(qd)
    base = None
    for mode in modes:
        rc, share = (mode.split("@") + ["1"])[:2]
        rc = "" if rc == "stream" else rc
        rep = GpuHierRep(op, recompute=rc, m2l_share=float(share))
        L, plan = rep._L, rep._plan
        s = torch.cuda.Stream()
        for _ in range(3):
            L.h2g_matvec(plan, qd.data_ptr(), out.data_ptr(), N, 1, 1, s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 20
        e0.record(s)
        for _ in range(it):
            L.h2g_matvec(plan, qd.data_ptr(), out.data_ptr(), N, 1, 1, s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        phi = out.cpu().numpy()
        if base is None:
            base = phi
        err = float(np.linalg.norm(phi - base) / np.linalg.norm(base))
        prof = rep.profile_phases(qd, out, iters=5)
        print(json.dumps({"mode": mode, "ms": ms, "matvec_per_s": 1e3 / ms,
                          "eff_TBps": (8 * op.mem_scalars + 16 * N) / ms * 1e-9,
                          "rel_vs_first": err, "launches": rep.launches_per_matvec(),
                          "phases_us": {p["phase"]: round(p["ms"] * 1e3, 1) for p in prof}}),
              flush=True)
        rep.close()


if __name__ == "__main__":
    main()
