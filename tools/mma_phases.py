"""Per-phase timing of the batched-RHS (DMMA) engine beside the single-RHS
streaming engine on the same operator (cfg 2 by default).  Diagnostics.

    python tools/mma_phases.py [N] [dim]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2309_14085_b200.builder import build_variant, uniform_points  # noqa: E402
from paper_2309_14085_b200.gpu_rep import GpuHierRep  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1048576
d = int(sys.argv[2]) if len(sys.argv) > 2 else 2
kern, eps = ("log2d", 1e-8) if d == 2 else ("lap3d", 1e-6)
op = build_variant("h2star-bt", uniform_points(N, d, 42), kern, 64, eps)
with GpuHierRep(op) as rep:
    q = torch.randn(N, dtype=torch.float64, device="cuda")
    phi = torch.empty_like(q)
    single = {r["phase"]: r for r in rep.profile_phases(q, phi, iters=10)}
    Q = torch.randn(N, 16, dtype=torch.float64, device="cuda")
    rep.matmat(Q)
    out = {"N": N, "dim": d, "lib": os.environ.get("H2G_LIB_PATH", "default"), "phases": []}
    for kb in (16, 8):
        tot = 0.0
        for r in rep.profile_phases_batched(kb, iters=10):
            s = single.get(r["phase"], {})
            fl = 2 * (r["bytes"] / 8) * kb
            tot += r["ms"]
            out["phases"].append({"kb": kb, "phase": r["phase"], "ms": round(r["ms"], 4),
                                  "ms_1rhs": round(s.get("ms", 0), 4),
                                  "GB": round(r["bytes"] / 1e9, 4),
                                  "tflops": round(fl / (r["ms"] * 1e-3) / 1e12, 2),
                                  "GBps": round(r["bytes"] / (r["ms"] * 1e-3) / 1e9, 1)})
        out[f"total_ms_kb{kb}"] = tot
    out["total_ms_1rhs"] = sum(r["ms"] for r in single.values())
print(json.dumps(out, indent=1))
