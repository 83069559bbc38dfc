"""Python API over the C-ABI (include/efem.h).  PyTorch provides device
memory and streams; every step of the assembly runs in libefem.so kernels.

    coords, elems = build_mesh(dim=3, n=64, jitter=0.15, seed=2)
    asm = Assembler(coords, elems, element=RT0)
    csr = asm.assemble()            # symbolic + numeric, CSR on the device
    dofs = asm.enumerate_dofs()     # dofs2nodes / elems2dofs / signs
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib

RT0, NED0 = _lib.EFEM_RT0, _lib.EFEM_NED0
MASS, STIFF, PATTERN, ALL = _lib.EFEM_MASS, _lib.EFEM_STIFF, _lib.EFEM_PATTERN, _lib.EFEM_ALL


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def launch_count() -> int:
    """Kernel launches issued by libefem.so since process start."""
    return int(_lib.load().efem_launch_count())


def mesh_sizes(dim: int, n: int):
    L = _lib.load()
    N, T = ctypes.c_int64(), ctypes.c_int64()
    _lib.check("efem_mesh_sizes", L.efem_mesh_sizes(dim, n, ctypes.byref(N), ctypes.byref(T)))
    return N.value, T.value


def build_mesh(dim: int, n: int, jitter: float, seed: int, device="cuda", stream=None):
    """Seeded structured mesh generated on the device (efem_build_mesh)."""
    N, T = mesh_sizes(dim, n)
    coords = torch.empty((N, dim), dtype=torch.float64, device=device)
    elems = torch.empty((T, dim + 1), dtype=torch.int32, device=device)
    with torch.cuda.device(coords.device):
        _lib.check("efem_build_mesh", _lib.load().efem_build_mesh(dim, n, jitter, seed, _ptr(coords), _ptr(elems),
                                                                 _stream(stream)))
    return coords, elems


@dataclass
class CSR:
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    vals_M: torch.Tensor
    vals_K: torch.Tensor

    @property
    def n_rows(self):
        return self.row_ptr.shape[0] - 1

    @property
    def nnz(self):
        return self.col_idx.shape[0]

    def as_torch(self, which="M"):
        v = self.vals_M if which == "M" else self.vals_K
        return torch.sparse_csr_tensor(self.row_ptr, self.col_idx, v, (self.n_rows, self.n_rows))


class Assembler:
    """One plan (efem_plan) for assembling `element` on a device mesh."""

    def __init__(self, coords: torch.Tensor, elems: torch.Tensor, element: int):
        if not coords.is_cuda or not elems.is_cuda:
            raise ValueError("coords / elems must be CUDA tensors")
        if coords.dtype != torch.float64 or elems.dtype != torch.int32:
            raise ValueError("coords must be float64, elems int32")
        self.coords = coords.contiguous()
        self.elems = elems.contiguous()
        self.dim = int(coords.shape[1])
        self.element = int(element)
        self.device = coords.device
        L = _lib.load()
        self._mesh = _lib.efem_mesh(self.dim, coords.shape[0], elems.shape[0], self.coords.data_ptr(),
                                    self.elems.data_ptr())
        plan = ctypes.c_void_p()
        ws = ctypes.c_size_t()
        _lib.check("efem_plan_create", L.efem_plan_create(ctypes.byref(plan), ctypes.byref(self._mesh),
                                                          self.element, ctypes.byref(ws)))
        self._plan = plan
        self.ws = torch.empty(max(int(ws.value), 256), dtype=torch.uint8, device=self.device)
        _lib.check("efem_plan_set_workspace", L.efem_plan_set_workspace(plan, _ptr(self.ws), self.ws.numel()))
        self.n_rows = None
        self.nnz = None

    @property
    def m(self):
        return 3 if self.dim == 2 else (4 if self.element == RT0 else 6)

    @property
    def ek(self):
        return 3 if (self.dim == 3 and self.element == RT0) else 2

    def close(self):
        if self._plan:
            _lib.load().efem_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def enumerate_dofs(self, stream=None):
        """dofs2nodes (R x 2|3), elems2dofs (T x m), signs (T x m int8)."""
        L = _lib.load()
        with torch.cuda.device(self.device):
            d = _lib.efem_dofs(0, None, None, None)
            _lib.check("efem_enumerate_dofs", L.efem_enumerate_dofs(self._plan, ctypes.byref(d), _stream(stream)))
            R = d.n_dofs
            T = self.elems.shape[0]
            d2n = torch.empty((R, self.ek), dtype=torch.int32, device=self.device)
            e2d = torch.empty((T, self.m), dtype=torch.int32, device=self.device)
            sg = torch.empty((T, self.m), dtype=torch.int8, device=self.device)
            d = _lib.efem_dofs(R, d2n.data_ptr() or None, e2d.data_ptr() or None, sg.data_ptr() or None)
            _lib.check("efem_enumerate_dofs", L.efem_enumerate_dofs(self._plan, ctypes.byref(d), _stream(stream)))
            return d2n, e2d, sg

    def symbolic(self, row_ptr: torch.Tensor | None = None, stream=None):
        L = _lib.load()
        R, nnz = ctypes.c_int64(), ctypes.c_int64()
        with torch.cuda.device(self.device):
            _lib.check("efem_assemble_symbolic", L.efem_assemble_symbolic(self._plan, ctypes.byref(R),
                                                                          ctypes.byref(nnz), _ptr(row_ptr),
                                                                          _stream(stream)))
        self.n_rows, self.nnz = R.value, nnz.value
        return self.n_rows, self.nnz

    def alloc_csr(self, n_rows=None, nnz=None) -> CSR:
        n_rows = self.n_rows if n_rows is None else n_rows
        nnz = self.nnz if nnz is None else nnz
        dev = self.device
        return CSR(torch.empty(n_rows + 1, dtype=torch.int32, device=dev),
                   torch.empty(nnz, dtype=torch.int32, device=dev),
                   torch.empty(nnz, dtype=torch.float64, device=dev),
                   torch.empty(nnz, dtype=torch.float64, device=dev))

    def _csr_struct(self, out: CSR):
        return _lib.efem_csr(self.n_rows, self.nnz, out.row_ptr.data_ptr(), out.col_idx.data_ptr(),
                             out.vals_M.data_ptr(), out.vals_K.data_ptr())

    def numeric(self, out: CSR, forms: int = ALL, stream=None):
        L = _lib.load()
        c = self._csr_struct(out)
        with torch.cuda.device(self.device):
            _lib.check("efem_assemble_numeric", L.efem_assemble_numeric(self._plan, forms, ctypes.byref(c),
                                                                        _stream(stream)))
        return out

    def check(self, stream=None):
        with torch.cuda.device(self.device):
            _lib.check("efem_plan_check", _lib.load().efem_plan_check(self._plan, _stream(stream)))

    def assemble(self, out: CSR | None = None, stream=None) -> CSR:
        """End to end from the device mesh: symbolic + numeric + check."""
        self.symbolic(stream=stream)
        if out is None or out.nnz != self.nnz or out.n_rows != self.n_rows:
            out = self.alloc_csr()
        self.numeric(out, ALL, stream=stream)
        self.check(stream=stream)
        return out

    def assemble_host(self, h_coords: torch.Tensor, h_elems: torch.Tensor, d_out: CSR, h_out: CSR, stream=None):
        """HOST mesh in -> HOST CSR out through efem_assemble_host (copies in
        the call).  Capacities of d_out / h_out must cover the pattern."""
        L = _lib.load()
        d = _lib.efem_csr(d_out.n_rows, d_out.nnz, d_out.row_ptr.data_ptr(), d_out.col_idx.data_ptr(),
                          d_out.vals_M.data_ptr(), d_out.vals_K.data_ptr())
        h = _lib.efem_csr(h_out.n_rows, h_out.nnz, h_out.row_ptr.data_ptr(), h_out.col_idx.data_ptr(),
                          h_out.vals_M.data_ptr(), h_out.vals_K.data_ptr())
        with torch.cuda.device(self.device):
            _lib.check("efem_assemble_host", L.efem_assemble_host(self._plan, _ptr(h_coords), _ptr(h_elems),
                                                                  ctypes.byref(d), ctypes.byref(h), _stream(stream)))
        self.n_rows, self.nnz = h.n_rows, h.nnz
        return h_out
