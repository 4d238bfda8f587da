"""Top SASS lines of an `ncu --page source --csv --print-source sass` dump by
warp-stall samples (per launch): the lines that hold the kernel."""
import csv
import sys


def main(path, top=40):
    with open(path, newline="") as fh:
        lines = fh.read().splitlines()
    blocks, cur = [], []
    for ln in lines:
        if ln.startswith('"Address"') or ln.startswith('"#"') or (ln.startswith('"') and "Source" in ln[:40]):
            if cur:
                blocks.append(cur)
            cur = [ln]
        elif cur:
            cur.append(ln)
    if cur:
        blocks.append(cur)
    for bi, blk in enumerate(blocks):
        rd = csv.reader(blk)
        hdr = next(rd)
        rows = [r for r in rd if len(r) == len(hdr)]
        key = None
        for k in ("Warp Stall Sampling (All Samples)", "Warp Stall Sampling (All Cycles)",
                  "Sampling Data (All)"):
            if k in hdr:
                key = k
                break
        if key is None:
            print(f"block {bi}: columns {hdr[:12]}")
            continue
        ki = hdr.index(key)
        si = hdr.index("Source") if "Source" in hdr else 1

        def val(r):
            try:
                return float(r[ki].replace(",", ""))
            except ValueError:
                return 0.0
        tot = sum(val(r) for r in rows) or 1.0
        print(f"== block {bi}: {len(rows)} lines, {tot:.0f} samples ({key})")
        extra = [c for c in hdr if "stall" in c.lower() and c != key][:0]
        for r in sorted(rows, key=val, reverse=True)[:top]:
            print(f"{100 * val(r) / tot:5.1f}%  {r[si][:110]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
