"""ncu evidence for bench.py's cfg-3 roofline (one GPU).

    python tools/ncu_cfg3.py build /tmp/cfg3     # native build (store="") -> export dir
    python tools/ncu_cfg3.py run /tmp/cfg3       # plain run: must exit 0 first
    ncu --set full --clock-control none --import-source on \
        -k regex:"stream_gemv|p2p_tasks" -s 32 -c 31 -o /tmp/prof_cfg3 \
        python tools/ncu_cfg3.py run /tmp/cfg3
    python tools/ncu_cfg3.py summarize /tmp/prof_cfg3.ncu-rep [out_dir]

The NCA pivot search (minutes) runs once, in ``build``, which exports
BASELINE configs[2] with only the transfer operators, pivots and points
(~1 GB); ``run`` re-evaluates the M2L / near blocks natively
(builder.materialize_blocks: bitwise the blocks of a stored build, seconds),
so the profiled command stays under ncu's 300 s plain-run limit.  It then
does 3 matvecs of the bench's headline plan (M2L evaluated at
bench.M2L_EVAL_SHARE, 16 filtered launches each) and 1 matvec of the
all-streamed plan (15 launches); -s 32 -c 31 captures the third headline
matvec and the streamed one.  ``summarize`` writes
traffic_cfg3_h2star-bt_eval.json / traffic_cfg3_h2star-bt.json (DRAM bytes
per matvec) and p2p_cfg3_h2star-bt.json (fp64-pipe utilisation of the P2P
launches, time-weighted).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _share():
    """Evaluated share of the M2L entries in the headline plan (bench.py's)."""
    sys.path.insert(0, ROOT)
    from bench import M2L_EVAL_SHARE
    return M2L_EVAL_SHARE
sys.path.insert(0, ROOT)

METRICS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active")


def build(path):
    from paper_2309_14085_b200.builder import build_variant, uniform_points
    op = build_variant("h2star-bt", uniform_points(1 << 20, 3, 42), "lap3d", 64, 1e-6,
                       store="")
    op.save_dir(path)


def run(path):
    import time
    import numpy as np
    sys.path.insert(0, ROOT)
    from bench import M2L_EVAL_SHARE
    from paper_2309_14085_b200.builder import materialize_blocks
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    from paper_2309_14085_b200.packed import PackedOperator
    t0 = time.time()
    op = materialize_blocks(PackedOperator.load_dir(path))  # = the stored build, bitwise
    print("materialized in", time.time() - t0, "s")
    q = np.random.default_rng(43).standard_normal(op.N)
    with GpuHierRep(op, recompute="m2l", m2l_share=M2L_EVAL_SHARE) as rep:
        for _ in range(3):
            rep.matvec(q)
        print("headline launches per matvec", rep.launches_per_matvec())
    with GpuHierRep(op) as rep:
        rep.matvec(q)
        print("streamed launches per matvec", rep.launches_per_matvec())


def _rows(rep_path):
    if rep_path.endswith(".csv"):  # an `ncu -i ... --page raw --csv` dump
        out = open(rep_path).read()
    else:
        out = subprocess.run(["ncu", "-i", rep_path, "--page", "raw", "--csv"], check=True,
                             capture_output=True, text=True).stdout
    lines = out.splitlines()
    rd = csv.reader(io.StringIO("\n".join(lines)))
    hdr = next(rd)
    units = next(rd)
    rows = []
    for r in rd:
        if len(r) != len(hdr):
            continue
        rows.append(dict(zip(hdr, r)))
    return rows, dict(zip(hdr, units))


def _f(r, k):
    v = r.get(k, "")
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def summarize(rep_path, n_head=16, out_dir=None):
    rows, units = _rows(rep_path)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
             "GB": 1e9}
    def by(r, k):
        return _f(r, k) * scale.get(units.get(k, "byte"), 1)
    tscale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9,
              "us": 1e-6, "ms": 1e-3, "s": 1.0}
    def t(r):
        return _f(r, "gpu__time_duration.sum") * tscale.get(units.get("gpu__time_duration.sum"), 1e-9)
    head, stream = rows[:n_head], rows[n_head:]
    out_dir = out_dir or os.path.join(ROOT, "profiles")
    os.makedirs(out_dir, exist_ok=True)
    for name, rr in (("traffic_cfg3_h2star-bt_eval.json", head),
                     ("traffic_cfg3_h2star-bt.json", stream)):
        rd = sum(by(r, "dram__bytes_read.sum") for r in rr)
        wr = sum(by(r, "dram__bytes_write.sum") for r in rr)
        out = {"config": "cfg3", "variant": "h2star-bt", "launches": len(rr),
               "mode": (f"M2L evaluated (share {_share():.1f}; the rest TMA-staged in the P2P tasks)"
                        if rr is head else "all streamed"),
               "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
               "kernel_time_s_serialised": sum(t(r) for r in rr),
               "per_launch": [{"kernel": r.get("Kernel Name", "")[:60], "us": t(r) * 1e6,
                               "dram_GB": (by(r, "dram__bytes_read.sum") + by(r, "dram__bytes_write.sum")) / 1e9,
                               "fp64_pipe_pct": _f(r, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")}
                              for r in rr],
               "note": "sum over the GEMV/P2P launches of ONE matvec (ncu --set full, "
                       "--clock-control none; cold-cache, serialised); tools/ncu_cfg3.py"}
        with open(os.path.join(out_dir, name), "w") as fh:
            json.dump(out, fh, indent=1)
        print(name, json.dumps({k: out[k] for k in ("launches", "dram_bytes_per_launch",
                                                   "kernel_time_s_serialised")}))
    p2p = [r for r in head if "p2p" in r.get("Kernel Name", "")]
    tt = sum(t(r) for r in p2p) or 1.0
    frac = sum(t(r) * _f(r, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
               for r in p2p) / tt / 100.0
    out = {"kernel": "p2p_tasks_kernel (M2L evaluated, cfg3 headline plan)", "launches": len(p2p),
           "time_s_serialised": tt, "fp64_pipe_frac": frac,
           "share_of_matvec_serialised": tt / (sum(t(r) for r in head) or 1.0),
           "metric": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active, "
                     "time-weighted over the P2P launches"}
    with open(os.path.join(out_dir, "p2p_cfg3_h2star-bt.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2])
    elif sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        summarize(sys.argv[2], out_dir=sys.argv[3] if len(sys.argv) > 3 else None)
