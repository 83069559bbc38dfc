"""Small driver for ncu: build the config's mesh, run the assembly step
`reps` times (profile with -s/-c to pick the launch).  --warm W: W
untimed steps first, then cudaProfilerStart (ncu --profile-from-start off
then captures the steady-state steps only: the fan pass's kernel choice
follows the previous step's read-back)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402
from workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--warm", type=int, default=0)
a = ap.parse_args()
C = CONFIGS[a.config]
coords, elems = api.build_mesh(C["dim"], C["n"], C["alpha"], C["seed"])
asm = api.Assembler(coords, elems, C["element"])
out = None
for _ in range(a.warm):
    out = asm.assemble(out)
torch.cuda.synchronize()
if a.warm:
    torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.reps):
    out = asm.assemble(out)
torch.cuda.synchronize()
print("ok", asm.n_rows, asm.nnz)
