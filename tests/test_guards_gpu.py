"""Out-of-bounds write guards (compute-sanitizer is closed on this GPU pool:
profiles/r2/compute_sanitizer_closed.log).  Every device buffer the library
writes -- the plan workspace, the CSR outputs, the DOF tables, the
distributed plans' slices -- is placed between canary zones filled with a
byte pattern; after symbolic + numeric, the asynchronous one-call form, the
DOF export and (2D) a distributed step, every canary must be intact.  Run
with EFEM_DEBUG_SYNC=1 the library also synchronises after every launch, so
an illegal access is reported at its launch site (tools/guard_run.sh)."""
import ctypes

import numpy as np
import pytest
import torch

from workloads import NED0, RT0

pytestmark = pytest.mark.gpu
PAD = 1 << 16  # bytes of canary on each side
PATTERN = 0xA5


class Guarded:
    """A device byte buffer [canary | payload | canary]."""

    def __init__(self, nbytes, device="cuda"):
        self.buf = torch.full((nbytes + 2 * PAD + 256,), PATTERN, dtype=torch.uint8, device=device)
        self.off = PAD + (-(self.buf.data_ptr() + PAD) % 256)  # 256-byte aligned payload
        self.n = nbytes

    def view(self, dtype, count):
        b = self.buf[self.off:self.off + count * torch.tensor([], dtype=dtype).element_size()]
        return b.view(dtype)

    def ptr(self):
        return self.buf.data_ptr() + self.off

    def intact(self):
        lo = self.buf[:self.off]
        hi = self.buf[self.off + self.n:]
        return bool((lo == PATTERN).all()) and bool((hi == PATTERN).all())


def _meshes(api, dim):
    from scipy.spatial import Delaunay

    yield api.build_mesh(dim, 5 if dim == 2 else 3, 0.2 if dim == 2 else 0.15, 1)
    yield api.build_mesh(dim, 37 if dim == 2 else 7, 0.2 if dim == 2 else 0.15, 2)
    rng = np.random.default_rng(dim)
    pts = np.concatenate([np.array(np.meshgrid(*[[0.0, 1.0]] * dim, indexing="ij")).reshape(dim, -1).T,
                          rng.random((300 if dim == 2 else 120, dim))])
    el = Delaunay(pts).simplices.astype(np.int32)
    x = pts[el]
    el = el[np.abs(np.linalg.det(x[:, 1:] - x[:, :1])) > 1e-9]
    yield torch.from_numpy(np.ascontiguousarray(pts)).cuda(), torch.from_numpy(np.ascontiguousarray(el)).cuda()


@pytest.mark.parametrize("dim,element", [(2, RT0), (2, NED0), (3, RT0), (3, NED0)],
                         ids=["rt0_2d", "ne0_2d", "rt0_3d", "ne0_3d"])
def test_canaries_intact(dim, element):
    from paper_1409_4618_b200 import _lib, api

    L = _lib.load()
    for coords, elems in _meshes(api, dim):
        asm = api.Assembler(coords, elems, element)
        ws = Guarded(asm.ws.numel())
        _lib.check("efem_plan_set_workspace", L.efem_plan_set_workspace(asm._plan, ctypes.c_void_p(ws.ptr()),
                                                                        asm.ws.numel()))
        asm.ws = None
        R, nnz = asm.symbolic()
        outs = [Guarded(4 * (R + 1)), Guarded(4 * nnz), Guarded(8 * nnz), Guarded(8 * nnz)]
        csr = api.CSR(outs[0].view(torch.int32, R + 1), outs[1].view(torch.int32, nnz),
                      outs[2].view(torch.float64, nnz), outs[3].view(torch.float64, nnz))
        asm.numeric(csr)
        asm.check()
        ref = [t.clone() for t in (csr.row_ptr, csr.col_idx, csr.vals_M, csr.vals_K)]
        asm.assemble_async(csr)
        asm.check()
        for a, b in zip(ref, (csr.row_ptr, csr.col_idx, csr.vals_M, csr.vals_K)):
            assert torch.equal(a, b)
        T, m = elems.shape[0], asm.m
        tabs = [Guarded(4 * R * asm.ek), Guarded(4 * T * m), Guarded(T * m)]
        d = _lib.efem_dofs(R, tabs[0].ptr(), tabs[1].ptr(), tabs[2].ptr())
        _lib.check("efem_enumerate_dofs", L.efem_enumerate_dofs(asm._plan, ctypes.byref(d), None))
        torch.cuda.synchronize()
        for g in [ws] + outs + tabs:
            assert g.intact()


def test_canaries_intact_distributed():
    from paper_1409_4618_b200 import api, dist

    coords, elems = api.build_mesh(2, 29, 0.2, 4)
    g = dist.DistGroup(coords, elems, RT0, dist.slab_bounds(elems.shape[0], 3))
    g.assemble()
    wins = g.last
    guards = []
    slices = []
    for w in wins:
        rows, nnz = w[1], w[3]
        gs = [Guarded(4 * (rows + 1)), Guarded(4 * nnz), Guarded(8 * nnz), Guarded(8 * nnz)]
        guards += gs
        slices.append(api.CSR(gs[0].view(torch.int32, rows + 1), gs[1].view(torch.int32, nnz),
                              gs[2].view(torch.float64, nnz), gs[3].view(torch.float64, nnz)))
    ref = g.concat()
    g.slices = slices
    g.assemble()
    got = g.concat()
    for a, b in zip(ref, got):
        assert a.tobytes() == b.tobytes()
    torch.cuda.synchronize()
    assert all(x.intact() for x in guards)
