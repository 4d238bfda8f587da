"""cfg-3 timing of one libh2g.so build variant (H2G_LIB_PATH) over M2L
evaluation shares, on an operator exported once (tools/ncu_cfg3.py build):

    python tools/ncu_cfg3.py build /tmp/cfg3
    H2G_LIB_PATH=.../libh2g_x.so python tools/variant_sweep.py /tmp/cfg3 0.7 0.6 0.5

One JSON line per share: ms per matvec (CUDA events, 20 matvecs after 5
warm-ups), the M2L phases' us, error vs the all-streamed result.  Diagnostics
only; bench.py is the measured contract.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2309_14085_b200.builder import materialize_blocks
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    from paper_2309_14085_b200.packed import PackedOperator
    op = materialize_blocks(PackedOperator.load_dir(sys.argv[1]))
    shares = [float(a) for a in sys.argv[2:]] or [0.7, 0.6]
    N = op.N
    q = np.random.default_rng(43).standard_normal(N)
    qd = torch.from_numpy(q).cuda()
    out = torch.empty_like(qd)
    base = None
    if os.environ.get("SWEEP_CHECK", "1") == "1":
        with GpuHierRep(op) as rep:
            base = rep.matvec(q)
    stream = torch.cuda.Stream()
    for sh in shares:
        with GpuHierRep(op, recompute="m2l", m2l_share=sh) as rep:
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
            phi = out.cpu().numpy()
            prof = rep.profile_phases(qd, out, iters=5)
            err = None if base is None else float(np.linalg.norm(phi - base) / np.linalg.norm(base))
            print(json.dumps({"lib": os.path.basename(os.environ.get("H2G_LIB_PATH", "libh2g.so")),
                              "share": sh, "ms": round(ms, 4), "err_vs_streamed": err,
                              "m2l_us": {p["phase"]: round(p["ms"] * 1e3, 1) for p in prof
                                         if p["phase"] in ("down_l3", "down_l4", "down_l5")}}),
                  flush=True)


if __name__ == "__main__":
    main()
