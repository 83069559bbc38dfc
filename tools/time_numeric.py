"""Time the numeric call alone (cold L2) for a config: median of reps."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402
from workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--reps", type=int, default=7)
a = ap.parse_args()
C = CONFIGS[a.config]
coords, elems = api.build_mesh(C["dim"], C["n"], C["alpha"], C["seed"])
asm = api.Assembler(coords, elems, C["element"])
out = asm.assemble()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for r in range(a.reps):
    flush.fill_(r)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    asm.numeric(out)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ts.sort()
print(f"config {a.config} ABL={os.environ.get('EFEM_NE3_ABL', '0')} numeric median {ts[len(ts)//2]:.3f} ms min {ts[0]:.3f}")
