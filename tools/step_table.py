"""Summarise an ncu per-kernel CSV (tools/step_profile.sh) as a table."""
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    d, order = {}, []
    for r in rows[1:]:
        k = (r[0], r[4].split("(")[0][-44:])
        if k not in d:
            d[k] = {}
            order.append(k)
        d[k][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    print(path)
    for k in order:
        m = d[k]
        print(f"  {k[1]:44s} {m['gpu__time_duration.sum'] / 1e3:9.1f} us  rd {m['dram__bytes_read.sum'] / 1e6:8.1f} MB"
              f"  wr {m['dram__bytes_write.sum'] / 1e6:8.1f} MB  inst {m['smsp__inst_executed.sum'] / 1e6:8.1f} M")
