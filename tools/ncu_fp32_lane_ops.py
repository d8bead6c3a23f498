"""Executed FP32 lane-ops per (pixel, control) pair from an ncu source page
(--page source --csv --print-source sass): packed FFMA2/FADD2/FMUL2 count two
lanes per thread instruction.  Validates bench.py's analytical roofline count."""
import csv
import re
import sys


def main(path, pixels, controls):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    i_s, i_t = hdr.index("Source"), hdr.index("Thread Instructions Executed")
    by = {}
    for r in data:
        m = re.match(r"(@!?P\d+\s+)?([A-Z0-9]+)", r[i_s].strip())
        if not m or not r[i_t].isdigit():
            continue
        op = m.group(2)
        mult = 2 if op in ("FFMA2", "FADD2", "FMUL2") else (1 if op in ("FFMA", "FADD", "FMUL") else 0)
        if mult:
            by[op] = by.get(op, 0) + mult * int(r[i_t])
    pairs = pixels * controls
    for op, v in sorted(by.items()):
        print(f"{op:6s} {v / pairs:8.3f} lane-ops per pair")
    print(f"total  {sum(by.values()) / pairs:8.3f} lane-ops per pair")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
