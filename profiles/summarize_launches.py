"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel
count, mean and total device time, and share of the total (cold-cache, serialised)."""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", ""))
            unit = r[ui]
            ms = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v if unit in ("ms", "msecond") else v / 1e6
            name = re.sub(r"\(.*", "", r[ki]).split("::")[-1]
            agg[name].append(ms)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':40s} {'n':>5s} {'mean_ms':>10s} {'total_ms':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:40]:40s} {len(v):5d} {sum(v)/len(v):10.4f} {sum(v):10.3f} {sum(v)/tot:7.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
