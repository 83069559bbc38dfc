"""B200 assembly times beside the paper's Tables 1 and 2
 at identical matrix sizes: the L-shape (0,1)^2 \\ (1/2,1)^2
(level L = the m = 2^(L+1) grid) and the unit cube (level L = the n = 6 2^(L-1)
Kuhn grid), unjittered like the paper's meshes.

    python examples/paper_tables.py [--lshape 5 .. 12] [--cube 1 .. 6] [--reps 5]

Per level and element: the end-to-end step (symbolic + numeric of both
matrices on one pattern, mesh already in HBM) and the numeric call restricted
to one matrix (K or M, pattern included), CUDA events, L2 flushed, median of
--reps.  The paper's times are MATLAB R2011b on 64 Xeon E7-8837 cores:
context, not a target.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402
from workloads import NED0, RT0  # noqa: E402


def timed(fn, flush, reps):
    ts = []
    for r in range(reps):
        flush.fill_(r & 0xff)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def level_times(c, e, element, flush, reps):
    asm = api.Assembler(c, e, element)
    out = asm.assemble()

    def step():
        asm.symbolic()
        asm.numeric(out, api.ALL)
        asm.check()

    t_step = timed(step, flush, reps)
    t_K = timed(lambda: asm.numeric(out, api.STIFF | api.PATTERN), flush, reps)
    t_M = timed(lambda: asm.numeric(out, api.MASS | api.PATTERN), flush, reps)
    size = asm.n_rows
    del asm, out
    torch.cuda.empty_cache()
    return size, t_step, t_K, t_M


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lshape", type=int, nargs="*", default=list(range(5, 13)))
    ap.add_argument("--cube", type=int, nargs="*", default=list(range(1, 7)))
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    P = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_counts.json")))["table1_2_times_s"]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    hdr = (f"{'level':>5} {'size':>11} | {'step RT':>9} {'K RT':>9} {'M RT':>9} | {'size':>11} {'step Ned':>9} "
           f"{'K Ned':>9} {'M Ned':>9} | paper K_RT M_RT K_Ned M_Ned (s)")
    print("Table 1 analogue: L-shape, 2D (seconds)\n" + hdr, flush=True)
    t1 = P["table1_lshape"]
    for L in a.lshape:
        c, e = api.build_lshape(2 ** (L + 1), 0.0, 0)
        sr, str_, kr, mr = level_times(c, e, RT0, flush, a.reps)
        sn, stn, kn, mn = level_times(c, e, NED0, flush, a.reps)
        i = t1["levels"].index(L) if L in t1["levels"] else None
        pp = f"{t1['K_RT'][i]} {t1['M_RT'][i]} {t1['K_Ned'][i]} {t1['M_Ned'][i]}" if i is not None else "-"
        print(f"{L:>5} {sr:>11} | {str_:>9.2e} {kr:>9.2e} {mr:>9.2e} | {sn:>11} {stn:>9.2e} {kn:>9.2e} {mn:>9.2e} | {pp}",
              flush=True)
        del c, e
        torch.cuda.empty_cache()
    print("\nTable 2 analogue: unit cube, 3D (seconds)\n" + hdr, flush=True)
    t2 = P["table2_cube"]
    for L in a.cube:
        c, e = api.build_mesh(3, 6 * 2 ** (L - 1), 0.0, 0)
        sr, str_, kr, mr = level_times(c, e, RT0, flush, a.reps)
        sn, stn, kn, mn = level_times(c, e, NED0, flush, a.reps)
        i = t2["levels"].index(L) if L in t2["levels"] else None
        pp = f"{t2['K_RT'][i]} {t2['M_RT'][i]} {t2['K_Ned'][i]} {t2['M_Ned'][i]}" if i is not None else "-"
        print(f"{L:>5} {sr:>11} | {str_:>9.2e} {kr:>9.2e} {mr:>9.2e} | {sn:>11} {stn:>9.2e} {kn:>9.2e} {mn:>9.2e} | {pp}",
              flush=True)
        del c, e
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
