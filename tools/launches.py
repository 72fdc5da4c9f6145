"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import csv
import sys
from collections import defaultdict


def main(path, steps=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(
                d.get("Metric Unit", "ns"), 1e-3)
            k = d["Kernel Name"][:80]
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    print(f"{'us total':>10} {'share':>6} {'n':>4}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1]:10.1f} {100 * v[1] / tot:5.1f}% {v[0]:4d}  {k}")
    print(f"{tot:10.1f}  total us")


if __name__ == "__main__":
    main(sys.argv[1])
