"""ncu driver for the batched-RHS (DMMA) engine: cfg2 operator, two 16-RHS
passes.  Diagnostics only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2309_14085_b200.builder import build_variant, uniform_points  # noqa: E402
from paper_2309_14085_b200.gpu_rep import GpuHierRep  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1048576
op = build_variant("h2star-bt", uniform_points(N, 2, 42), "log2d", 64, 1e-8)
with GpuHierRep(op) as rep:
    Q = torch.randn(N, 16, dtype=torch.float64, device="cuda")
    for _ in range(2):
        rep.matmat(Q)
    torch.cuda.synchronize()
print("done")
