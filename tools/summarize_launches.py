"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel count, total/mean device time and share (cold-cache, serialised)."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def us(d):
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    return v / 1000 if u in ("ns", "nsecond") else (v * 1000 if u in ("ms", "msecond") else v)


def main(path):
    data = load(path)
    agg = collections.OrderedDict()
    for d in data:
        name = re.sub(r"\(.*", "", d["Kernel Name"])
        name = re.sub(r"cub::(\w+)<.*", r"cub::\1", name)[:70]
        agg.setdefault(name, []).append(us(d))
    total = sum(sum(v) for v in agg.values())
    print(f"# {path}: {len(data)} launches, {total / 1000:.1f} ms total device time (serialised, cold cache)")
    print(f"{'kernel':70s} {'n':>6s} {'total_ms':>10s} {'mean_us':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:70s} {len(v):6d} {sum(v) / 1000:10.2f} {sum(v) / len(v):10.1f} {sum(v) / total:7.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
