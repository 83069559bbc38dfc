"""profiles/traffic.json from the per-kernel step captures (tools/profile_step.py under
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,...): per config the DRAM
bytes of one whole assembly step (all kernels but the untimed mesh generator),
read and write separately, and per kernel.  bench.py reports them as the
roofline's static `traffic`.  Usage: python tools/traffic_json.py <dir with step_cfg*.csv>"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import CONFIGS  # noqa: E402

d = sys.argv[1]
out = {"_doc": "DRAM bytes (dram__bytes_read.sum / dram__bytes_write.sum) of one assembly step per config, "
               "summed over its kernels (mesh generation excluded), from ncu captures of tools/profile_step.py "
               "(cold L2, serialised launches): a static capture read by bench.py"}
for c in (2, 3, 4, 5):
    path = os.path.join(d, f"step_cfg{c}.csv")
    if not os.path.exists(path):
        continue
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    per, order = {}, []
    for r in rows[1:]:
        k = (r[0], r[h.index("Kernel Name")].split("(")[0])
        if k not in per:
            per[k] = {}
            order.append(k)
        per[k][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    kern = []
    for k in order:
        if "k_coords" in k[1] or "k_elems" in k[1]:
            continue
        m = per[k]
        kern.append({"kernel": k[1][-60:], "us": m["gpu__time_duration.sum"] / 1e3,
                     "dram_read": int(m["dram__bytes_read.sum"]), "dram_write": int(m["dram__bytes_write.sum"])})
    out[CONFIGS[c]["name"]] = {
        "step_dram_read": sum(x["dram_read"] for x in kern), "step_dram_write": sum(x["dram_write"] for x in kern),
        "step_dram_bytes": sum(x["dram_read"] + x["dram_write"] for x in kern),
        "source": f"profiles/r2/step_cfg{c}.csv", "kernels": kern}
print(json.dumps(out, indent=1))
