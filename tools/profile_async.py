"""ncu target: the bench step (efem_assemble_async after one symbolic call) of a config, `reps` times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402
from workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
C = CONFIGS[a.config]
coords, elems = api.build_mesh(C["dim"], C["n"], C["alpha"], C["seed"])
asm = api.Assembler(coords, elems, C["element"])
asm.symbolic()
out = asm.alloc_csr()
for _ in range(a.reps):
    asm.assemble_async(out)
    asm.check()
torch.cuda.synchronize()
print("ok")
