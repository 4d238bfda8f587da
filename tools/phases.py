"""Per-phase single-RHS timing (CUDA events) of one variant on a BASELINE-shaped
operator.  Diagnostics.

    python tools/phases.py [variant] [N] [dim]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2309_14085_b200.builder import build_variant, uniform_points  # noqa: E402
from paper_2309_14085_b200.gpu_rep import GpuHierRep, schedule_info  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "h2plusH-star"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1048576
d = int(sys.argv[3]) if len(sys.argv) > 3 else 2
kern, eps = ("log2d", 1e-8) if d == 2 else ("lap3d", 1e-6)
op = build_variant(variant, uniform_points(N, d, 42), kern, 64, eps)
info = {p["name"]: p for p in schedule_info(op)["phases"]}
with GpuHierRep(op) as rep:
    q = torch.randn(N, dtype=torch.float64, device="cuda")
    phi = torch.empty_like(q)
    rows = rep.profile_phases(q, phi, iters=20)
out = []
for r in rows:
    i = info.get(r["phase"], {})
    out.append({"phase": r["phase"], "us": round(r["ms"] * 1e3, 1), "GB": round(r["bytes"] / 1e9, 4),
                "GBps": round(r["bytes"] / max(r["ms"], 1e-9) / 1e6, 1), "tasks": i.get("tasks"),
                "chunks": i.get("chunks"), "ctas": i.get("ctas"),
                "max_cta_MB": round(i.get("max_cta_bytes", 0) / 1e6, 3)})
print(json.dumps({"variant": variant, "N": N, "dim": d, "total_us": round(sum(o["us"] for o in out), 1),
                  "phases": out}, indent=1))
