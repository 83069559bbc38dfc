"""Tiny end-to-end call for compute-sanitizer runs:
    python tools/tiny.py dim element n        structured mesh (n cells per axis)
    python tools/tiny.py dl2|dl3 element 0    scipy Delaunay mesh of seeded points
Runs symbolic + numeric + check, the asynchronous one-call form, and the
DOF-table export."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1409_4618_b200 import api  # noqa: E402

kind, element, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
if kind.startswith("dl"):
    from scipy.spatial import Delaunay

    dim = int(kind[2])
    rng = np.random.default_rng(7)
    pts = np.concatenate([np.array(np.meshgrid(*[[0.0, 1.0]] * dim, indexing="ij")).reshape(dim, -1).T,
                          rng.random((400 if dim == 2 else 150, dim))])
    el = Delaunay(pts).simplices.astype(np.int32)
    x = pts[el]
    el = el[np.abs(np.linalg.det(x[:, 1:] - x[:, :1])) > 1e-9]
    coords = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    elems = torch.from_numpy(np.ascontiguousarray(el)).cuda()
else:
    dim = int(kind)
    coords, elems = api.build_mesh(dim, n, 0.2 if dim == 2 else 0.15, 5)
asm = api.Assembler(coords, elems, element)
out = asm.assemble()
asm.enumerate_dofs()
asm.assemble_async(out)
asm.check()
torch.cuda.synchronize()
print("ok", asm.n_rows, asm.nnz)
