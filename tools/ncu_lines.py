"""Per-source-line instructions and stall samples of an ncu report:
python tools/ncu_lines.py <rep> [file substring] [min share]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ".cu"
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = fil = None
agg, samp, txt = collections.Counter(), collections.Counter(), {}
for r in rows:
    if r and r[0] == "File Path":
        fil = r[1].split("/")[-1]
        continue
    if len(r) < 9 or r[0] == "Line No":
        continue
    if r[0] != "":
        cur = (fil, int(r[0]))
        txt[cur] = r[1].strip()[:100]
        continue
    try:
        n, s = int(r[7]), int(r[4])
    except ValueError:
        continue
    agg[cur] += n
    samp[cur] += s
tot, ts = sum(agg.values()), max(1, sum(samp.values()))
print("instructions", tot, "samples", ts)
for k in sorted(agg, key=lambda k: (k[0], k[1])):
    if want in k[0] and (agg[k] > mn * tot or samp[k] > mn * ts):
        print(f"{k[0][:14]:14s}{k[1]:5d} {100 * agg[k] / tot:5.1f}% s{100 * samp[k] / ts:5.1f}%  {txt[k]}")
