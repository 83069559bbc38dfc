"""Per-source-line instruction / stall shares of one kernel in an ncu report."""
import csv
import subprocess
import sys


def main(path, kernel, top=25):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", "regex:" + kernel,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hi]
    ie, iss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    lines = []
    for r in rows[hi + 1:]:
        if r and r[0] != "" and len(r) > max(ie, iss):
            try:
                lines.append((int(r[ie] or 0), int(r[iss] or 0), r[0], r[1][:100]))
            except ValueError:
                pass
    tot = sum(x[0] for x in lines) or 1
    tots = sum(x[1] for x in lines) or 1
    print(f"total warp instructions {tot}, stall samples {tots}")
    for x in sorted(lines, key=lambda x: -x[1])[:top]:
        print(f"{100 * x[0] / tot:5.1f}% inst {100 * x[1] / tots:5.1f}% stall  L{x[2]}: {x[3]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)


def by_file(path, kernel):
    """Instruction totals per source file (cuda view)."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", "regex:" + kernel,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    out = {}
    cur = None
    rows = list(csv.reader(raw.splitlines()))
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
    return out
