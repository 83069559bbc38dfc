"""Time the numeric and symbolic calls alone (cold L2) for a config: median of reps."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402
from workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--reps", type=int, default=9)
ap.add_argument("--tag", default="")
a = ap.parse_args()
C = CONFIGS[a.config]
coords, elems = api.build_mesh(C["dim"], C["n"], C["alpha"], C["seed"])
asm = api.Assembler(coords, elems, C["element"])
out = asm.assemble()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn):
    ts = []
    for r in range(a.reps):
        flush.fill_(r)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2], ts[0]


sm, smin = timed(lambda: asm.symbolic())
nm, nmin = timed(lambda: asm.numeric(out))
print(f"config {a.config} {a.tag} symbolic median {sm:.4f} ms (min {smin:.4f})  numeric median {nm:.4f} ms (min {nmin:.4f})")
