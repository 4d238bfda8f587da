"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every engine and protocol on tiny golden operators, results checked against
the reference's own matvec.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Covers: the TMA-bulk streaming engine (owned and split phases, PDL between
phases, byte ring / record ring / mbarriers), the batched DMMA engine (k-split
and group mode), the P2P kernel-evaluation engine (dynamic task counter and
its reset), hybrid phases (both engines concurrently), sharded virtual ranks
(pack / unpack / x halo), and the pinned host-call graph.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def check(name, phi, ref, tol=1e-12):
    e = float(np.linalg.norm(np.asarray(phi) - ref) / np.linalg.norm(ref))
    print(f"{name}: rel err {e:.2e}", flush=True)
    assert e <= tol, (name, e)


def main():
    import torch
    from golden_io import load_golden
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    from paper_2309_14085_b200.sharded import ShardedGpuHierRep
    for name in ("g2d_log_h2star", "g3d_lap_h2plusH"):
        op, z, meta = load_golden(name)
        with GpuHierRep(op) as rep:
            check(f"{name} stream", rep.matvec(z["q"]), z["phi_ref"])
            Q = np.repeat(z["Q"], 8, axis=1)  # 16 RHS: batched DMMA engine
            P = rep.matmat(Q)
            check(f"{name} dmma16", P[:, 0], z["Phi_ref"][:, 0])
            q_pin = torch.from_numpy(z["q"]).pin_memory().numpy()
            out = torch.empty(op.N, dtype=torch.float64).pin_memory().numpy()
            rep.matvec(q_pin, out=out)
            check(f"{name} pinned graph", out, z["phi_ref"])
        os.environ["H2G_MMA_GROUP_MIN_TASKS"] = "1"
        with GpuHierRep(op) as rep:
            check(f"{name} dmma group", rep.matmat(np.tile(z["Q"], (1, 4)))[:, 1], z["Phi_ref"][:, 1])
        os.environ.pop("H2G_MMA_GROUP_MIN_TASKS")
        with GpuHierRep(op, recompute="near,m2l") as rep:
            check(f"{name} p2p", rep.matvec(z["q"]), z["phi_ref"])
            check(f"{name} p2p again", rep.matvec(z["q"]), z["phi_ref"])
        os.environ["H2G_M2L_STREAM_SHARE"] = "0.4"
        with GpuHierRep(op, recompute="m2l") as rep:
            check(f"{name} hybrid", rep.matvec(z["q"]), z["phi_ref"])
        os.environ.pop("H2G_M2L_STREAM_SHARE")
        R = 2
        reps = [ShardedGpuHierRep(op, r, R, device=0) for r in range(R)]
        qd = torch.from_numpy(z["q"]).cuda()
        s = torch.cuda.current_stream().cuda_stream
        mx = max(1, reps[0].info["max_send_slots"])
        recv = torch.zeros(mx * R, dtype=torch.float64, device="cuda")
        for r, rp in enumerate(reps):
            send = torch.zeros(mx, dtype=torch.float64, device="cuda")
            rp.begin(qd, s)
            rp.pack(send, s)
            recv[r * mx:(r + 1) * mx] = send
        phi = torch.zeros_like(qd)
        for rp in reps:
            part = torch.zeros_like(qd)
            rp.unpack(recv, s)
            rp.end(part, s)
            phi += part
        torch.cuda.synchronize()
        check(f"{name} sharded x{R}", phi.cpu().numpy(), z["phi_ref"])
        for rp in reps:
            rp.close()
    print("SANITIZE_CASES_OK")


if __name__ == "__main__":
    main()
