"""Print the key metrics of every kernel in an ncu report (raw page)."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def main(path, top_stalls=6):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    for d in data:
        name = d[hdr.index("Kernel Name")].split("(")[0]
        print("==", name)
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"   {w}: {d[i]} {units[i]}")
        st = [(h, d[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
              and h.endswith("_per_issue_active.ratio")]
        st = sorted(st, key=lambda x: -float(x[1].replace(",", "") or 0))[:top_stalls]
        print("   stalls:", ", ".join(f"{h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]}={float(v):.2f}" for h, v in st))


if __name__ == "__main__":
    main(sys.argv[1])
