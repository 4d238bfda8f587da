"""DRAM traffic of one matvec, for bench.py's roofline.traffic.

Run under ncu (one GPU):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --print-units base --clock-control none -k regex:"stream_gemv|p2p_tasks" --csv \
      --log-file gpurun_out/traffic.csv python tools/ncu_traffic.py cfg2 [recompute]
then  python tools/ncu_traffic.py --summarize gpurun_out/traffic.csv cfg2 h2star-bt
writes profiles/traffic_<cfg>_<variant>.json (sum over the LAST matvec's launches).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PRESETS = {"cfg2": (1048576, 2, "log2d", 1e-8), "cfg3": (1048576, 3, "lap3d", 1e-6)}


def run(cfg, recompute=""):
    import numpy as np
    from paper_2309_14085_b200.builder import build_variant, uniform_points
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    N, d, k, eps = PRESETS[cfg]
    op = build_variant("h2star-bt", uniform_points(N, d, 42), k, 64, eps)
    q = np.random.default_rng(43).standard_normal(N)
    with GpuHierRep(op, recompute=recompute) as rep:
        for _ in range(2):
            rep.matvec(q)
        print("launches_per_matvec", rep.launches_per_matvec())


def summarize(path, cfg, variant, per_matvec):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    by_id = {}
    for r in rows:
        by_id.setdefault(r["ID"], {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        by_id[r["ID"]]["name"] = r["Kernel Name"]
    ids = sorted(by_id, key=int)[-per_matvec:]
    tot_r = sum(by_id[i]["dram__bytes_read.sum"] for i in ids)
    tot_w = sum(by_id[i]["dram__bytes_write.sum"] for i in ids)
    unit = 1.0
    out = {"config": cfg, "variant": variant, "launches": len(ids),
           "dram_bytes_read": tot_r * unit, "dram_bytes_write": tot_w * unit,
           "dram_bytes_per_launch": (tot_r + tot_w) * unit,
           "note": "sum over the GEMV launches of ONE matvec (the roofline's 'achieved' also "
                   "aggregates all GEMV phases of one matvec); ncu --metrics dram__bytes_*"}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    suffix = "_eval" if len(sys.argv) > 6 and sys.argv[6] else ""
    with open(os.path.join(ROOT, "profiles", f"traffic_{cfg}_{variant}{suffix}.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1] == "--summarize":
        summarize(sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5]))
    else:
        run(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
