"""Per-region instruction / stall shares from `ncu -i rep --page source --csv --print-source sass`."""
import csv
import sys


def main(path, width=32, thresh=0.01):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    i_s, i_w, i_e = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    num = lambda v: int(v) if v.isdigit() else 0
    te = sum(num(r[i_e]) for r in data) or 1
    tw = sum(num(r[i_w]) for r in data) or 1
    for b in range(0, len(data), width):
        blk = data[b:b + width]
        e = sum(num(r[i_e]) for r in blk)
        w = sum(num(r[i_w]) for r in blk)
        if e / te > thresh or w / tw > thresh:
            top = max(blk, key=lambda r: num(r[i_w]))
            print(f"{b:6d} exec {100 * e / te:5.1f}%  stall {100 * w / tw:5.1f}%  top: {top[i_s].strip()[:60]}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(a) for a in sys.argv[2:3]))


def reasons(path, lo, hi):
    """Stall-reason totals over SASS rows [lo, hi)."""
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = [hdr.index(c) for c in cols]
    tot = [sum(int(r[i]) if r[i].isdigit() else 0 for r in data[lo:hi]) for i in idx]
    s = sum(tot) or 1
    return sorted(((c, t / s) for c, t in zip(cols, tot) if t), key=lambda x: -x[1])
