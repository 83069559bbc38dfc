"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1000.0 if u in ("ns", "nsecond") else (v * 1000.0 if u in ("ms", "msecond") else v)
        agg.setdefault(r[ki].split("(")[0][:80], []).append(v)
    out = []
    for k, v in agg.items():
        out.append((k, len(v), sum(v) / len(v)))
    return out


if __name__ == "__main__":
    for k, n, us in summarize(sys.argv[1]):
        print(f"{n:5d} x {us:10.1f} us  {k}")
