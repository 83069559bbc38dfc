"""Tiny end-to-end call for compute-sanitizer runs: python tools/tiny.py dim element n"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402

dim, element, n = (int(x) for x in sys.argv[1:4])
coords, elems = api.build_mesh(dim, n, 0.2 if dim == 2 else 0.15, 5)
asm = api.Assembler(coords, elems, element)
out = asm.assemble()
torch.cuda.synchronize()
print("ok", asm.n_rows, asm.nnz)
