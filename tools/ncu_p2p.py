"""Small driver for ncu captures of the P2P engine: one 3D 1/r operator,
a few matvecs with the evaluated near + M2L path.  Diagnostics only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
mode = sys.argv[2] if len(sys.argv) > 2 else "near,m2l"
share = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0  # m2l_recompute_share
from paper_2309_14085_b200.builder import build_variant, uniform_points  # noqa: E402
from paper_2309_14085_b200.gpu_rep import GpuHierRep  # noqa: E402

op = build_variant("h2star-bt", uniform_points(N, 3, 42), "lap3d", 64, 1e-6)
q = np.random.default_rng(43).standard_normal(N)
with GpuHierRep(op, recompute=mode, m2l_share=share) as rep:
    for _ in range(3):
        rep.matvec(q)
print("done", N, mode)
