"""One-kernel ncu report: issue / occupancy, top stalls and the
instruction mix by opcode (share of instructions / of stall samples).
    python tools/ncu_mix.py <rep.ncu-rep> ..."""
import collections
import csv
import io
import subprocess
import sys


def page(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    r = page(rep, "--page", "raw", "--csv")
    h, v = r[0], r[2]
    g = dict(zip(h, v))
    def f(k):
        try:
            return float(g[k].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")
    print("time us", f("gpu__time_duration.sum") / 1e3,
          " dram rd MB", f("dram__bytes_read.sum") / 1e6, " wr MB", f("dram__bytes_write.sum") / 1e6)
    for k in ("sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "smsp__inst_executed.sum",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__occupancy_limit_shared_mem",
              "launch__occupancy_limit_registers", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"):
        print(" ", k, g.get(k))
    st = []
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            st.append((f(k), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
    print("  stalls:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:7]))
    rows = page(rep, "--page", "source", "--csv", "--print-source", "sass")
    hh = rows[1]
    I, S, src = hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
    ops, samp = collections.Counter(), collections.Counter()
    for x in rows[2:]:
        if len(x) <= I:
            continue
        toks = x[src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        ops[op] += int(x[I] or 0)
        samp[op] += int(x[S] or 0)
    tot, ts = sum(ops.values()), max(1, sum(samp.values()))
    print("  inst", tot, ":", ", ".join(f"{o} {100 * n / tot:.1f}%/{100 * samp[o] / ts:.0f}%s" for o, n in ops.most_common(14)))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(rep)
        main(rep)
