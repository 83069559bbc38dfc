"""One call of each f-row kernel on config 2's mesh (the ncu target for
tools/f_rows_bench.py's table)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402
from workloads import CONFIGS  # noqa: E402

C = CONFIGS[2]
coords, elems = api.build_mesh(2, C["n"], C["alpha"], C["seed"], device="cuda:0")
asm = api.Assembler(coords, elems, C["element"])
A = asm.assemble()
T = elems.shape[0]
F = torch.randn((T, 12, 2), dtype=torch.float64, device="cuda")
D = torch.randn((T, 12, 1), dtype=torch.float64, device="cuda")
u = torch.randn(asm.n_rows, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
api.quad_points(coords, elems)
asm.load(F, api.VALUE)
api.norm_l2(coords, elems, F)
asm.field_error(u, F, D)
api.spmv(A, u)
torch.cuda.synchronize()
