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


def build_lshape(m: int, jitter: float = 0.0, seed: int = 0, device="cuda", stream=None):
    """The paper's 2D timing domain (0,1)^2 minus (1/2,1)^2 on the m x m grid (m even)."""
    L = _lib.load()
    N, T = ctypes.c_int64(), ctypes.c_int64()
    _lib.check("efem_lshape_sizes", L.efem_lshape_sizes(m, ctypes.byref(N), ctypes.byref(T)))
    coords = torch.empty((N.value, 2), dtype=torch.float64, device=device)
    elems = torch.empty((T.value, 3), dtype=torch.int32, device=device)
    with torch.cuda.device(coords.device):
        _lib.check("efem_build_mesh_lshape", L.efem_build_mesh_lshape(m, jitter, seed, _ptr(coords), _ptr(elems),
                                                                      _stream(stream)))
    return coords, elems


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

    def set_exact(self, exact: bool = True):
        """NE0 3D: exact edge-row sizes for non-manifold meshes (slower symbolic)."""
        _lib.check("efem_plan_set_exact", _lib.load().efem_plan_set_exact(self._plan, int(bool(exact))))
        self.n_rows = self.nnz = None

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

    def assemble_async(self, out: CSR, forms: int = ALL, stream=None) -> CSR:
        """The whole hot path without a host round trip into an `out` sized by
        an earlier symbolic call (capacities); follow with check()."""
        c = _lib.efem_csr(out.n_rows, out.nnz, out.row_ptr.data_ptr(), out.col_idx.data_ptr(),
                          out.vals_M.data_ptr(), out.vals_K.data_ptr())
        with torch.cuda.device(self.device):
            _lib.check("efem_assemble_async", _lib.load().efem_assemble_async(self._plan, forms, ctypes.byref(c),
                                                                              _stream(stream)))
        return out

    def check(self, stream=None):
        with torch.cuda.device(self.device):
            _lib.check("efem_plan_check", _lib.load().efem_plan_check(self._plan, _stream(stream)))

    def check_async(self, stream=None):
        """Enqueue the flag / size read-back of check() without waiting."""
        with torch.cuda.device(self.device):
            _lib.check("efem_plan_check_async", _lib.load().efem_plan_check_async(self._plan, _stream(stream)))

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


# --------------------------------------------------------------------------- f1 / f2: vectorized integration
VALUE, DERIVATIVE = _lib.EFEM_PAIR_VALUE, _lib.EFEM_PAIR_DERIV


def quad_size(dim: int) -> int:
    """Points per element of the degree-6 rule (12 triangles, 24 tetrahedra)."""
    return _lib.load().efem_quad_size(dim)


def _mesh_struct(coords: torch.Tensor, elems: torch.Tensor):
    return _lib.efem_mesh(int(coords.shape[1]), coords.shape[0], elems.shape[0], coords.data_ptr(),
                          elems.data_ptr())


def quad_points(coords: torch.Tensor, elems: torch.Tensor, stream=None) -> torch.Tensor:
    """Physical quadrature points F_K(xh_q) of every element: (T, nq, dim)."""
    dim = int(coords.shape[1])
    pts = torch.empty((elems.shape[0], quad_size(dim), dim), dtype=torch.float64, device=coords.device)
    m = _mesh_struct(coords, elems)
    with torch.cuda.device(coords.device):
        _lib.check("efem_quad_points", _lib.load().efem_quad_points(ctypes.byref(m), _ptr(pts), _stream(stream)))
    return pts


def norm_l2(coords: torch.Tensor, elems: torch.Tensor, fq: torch.Tensor, stream=None):
    """(total, per_element) of sum_K sum_q w |det| |f|^2 for f values (T, nq[, nf])."""
    fq = fq.contiguous()
    nf = 1 if fq.dim() == 2 else int(fq.shape[2])
    L = _lib.load()
    m = _mesh_struct(coords, elems)
    ws_bytes = ctypes.c_size_t()
    per = torch.empty(elems.shape[0], dtype=torch.float64, device=coords.device)
    tot = torch.empty(1, dtype=torch.float64, device=coords.device)
    with torch.cuda.device(coords.device):
        _lib.check("efem_norm_l2", L.efem_norm_l2(ctypes.byref(m), None, nf, None, None, None, ctypes.byref(ws_bytes),
                                                  _stream(stream)))
        ws = torch.empty(int(ws_bytes.value), dtype=torch.uint8, device=coords.device)
        _lib.check("efem_norm_l2", L.efem_norm_l2(ctypes.byref(m), _ptr(fq), nf, _ptr(per), _ptr(tot), _ptr(ws),
                                                  ctypes.byref(ws_bytes), _stream(stream)))
    return tot, per


def _assembler_load(self, fq: torch.Tensor, pairing: int = VALUE, stream=None) -> torch.Tensor:
    """Load vector against the global basis (after symbolic): (n_dofs,)."""
    if self.n_rows is None:
        self.symbolic(stream=stream)
    fq = fq.contiguous()
    b = torch.empty(self.n_rows, dtype=torch.float64, device=self.device)
    with torch.cuda.device(self.device):
        _lib.check("efem_assemble_load", _lib.load().efem_assemble_load(self._plan, pairing, _ptr(fq), _ptr(b),
                                                                        _stream(stream)))
    return b


def _assembler_field_error(self, coeffs: torch.Tensor, Eq: torch.Tensor, Dq: torch.Tensor, stream=None):
    """Device tensor [||E - v||^2, ||D E - D v||^2] for v = sum_i coeffs_i phi_i."""
    L = _lib.load()
    ws_bytes = ctypes.c_size_t()
    err = torch.empty(2, dtype=torch.float64, device=self.device)
    Eq, Dq, coeffs = Eq.contiguous(), Dq.contiguous(), coeffs.contiguous()
    with torch.cuda.device(self.device):
        _lib.check("efem_field_error", L.efem_field_error(self._plan, None, None, None, None, None,
                                                          ctypes.byref(ws_bytes), _stream(stream)))
        ws = torch.empty(max(int(ws_bytes.value), 8), dtype=torch.uint8, device=self.device)
        _lib.check("efem_field_error", L.efem_field_error(self._plan, _ptr(coeffs), _ptr(Eq), _ptr(Dq), _ptr(err),
                                                          _ptr(ws), ctypes.byref(ws_bytes), _stream(stream)))
    return err


Assembler.load = _assembler_load
Assembler.field_error = _assembler_field_error


def _csr_ptrs(A: CSR):
    return _lib.efem_csr(A.n_rows, A.nnz, A.row_ptr.data_ptr(), A.col_idx.data_ptr(), A.vals_M.data_ptr(),
                         A.vals_K.data_ptr())


def spmv(A: CSR, x: torch.Tensor, alpha: float = 1.0, beta: float = 1.0, stream=None) -> torch.Tensor:
    """y = alpha K x + beta M x."""
    y = torch.empty_like(x)
    c = _csr_ptrs(A)
    with torch.cuda.device(x.device):
        _lib.check("efem_spmv", _lib.load().efem_spmv(ctypes.byref(c), alpha, beta, _ptr(x), _ptr(y),
                                                      _stream(stream)))
    return y


def cg(A: CSR, b: torch.Tensor, alpha: float = 1.0, beta: float = 1.0, x0: torch.Tensor | None = None,
       rtol: float = 1e-12, maxit: int = 100000, stream=None):
    """Jacobi-preconditioned CG for (alpha K + beta M) x = b; returns (x, iters, relres)."""
    L = _lib.load()
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    c = _csr_ptrs(A)
    ws_bytes = ctypes.c_size_t()
    it, rr = ctypes.c_int(), ctypes.c_double()
    with torch.cuda.device(b.device):
        _lib.check("efem_cg", L.efem_cg(ctypes.byref(c), alpha, beta, None, None, rtol, maxit, ctypes.byref(it),
                                        ctypes.byref(rr), None, ctypes.byref(ws_bytes), _stream(stream)))
        ws = torch.empty(int(ws_bytes.value), dtype=torch.uint8, device=b.device)
        _lib.check("efem_cg", L.efem_cg(ctypes.byref(c), alpha, beta, _ptr(b), _ptr(x), rtol, maxit,
                                        ctypes.byref(it), ctypes.byref(rr), _ptr(ws), ctypes.byref(ws_bytes),
                                        _stream(stream)))
    return x, it.value, rr.value


# --------------------------------------------------------------------------- f3: P1 nodal elements
class P1Assembler:
    """P1 (nodal) Laplacian stiffness / mass / load on a device mesh (efem_p1_plan)."""

    def __init__(self, coords: torch.Tensor, elems: torch.Tensor):
        self.coords, self.elems = coords.contiguous(), elems.contiguous()
        self.device = coords.device
        L = _lib.load()
        self._mesh = _mesh_struct(self.coords, self.elems)
        plan = ctypes.c_void_p()
        ws = ctypes.c_size_t()
        _lib.check("efem_p1_plan_create", L.efem_p1_plan_create(ctypes.byref(plan), ctypes.byref(self._mesh),
                                                                ctypes.byref(ws)))
        self._plan = plan
        self.ws = torch.empty(max(int(ws.value), 256), dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check("efem_p1_plan_set_workspace", L.efem_p1_plan_set_workspace(plan, _ptr(self.ws),
                                                                                  self.ws.numel()))
        self.n_rows = self.nnz = None

    def __del__(self):
        try:
            if self._plan:
                _lib.load().efem_p1_plan_destroy(self._plan)
                self._plan = None
        except Exception:
            pass

    def assemble(self, stream=None) -> CSR:
        L = _lib.load()
        R, nnz = ctypes.c_int64(), ctypes.c_int64()
        with torch.cuda.device(self.device):
            _lib.check("efem_p1_symbolic", L.efem_p1_symbolic(self._plan, ctypes.byref(R), ctypes.byref(nnz),
                                                              _stream(stream)))
            self.n_rows, self.nnz = R.value, nnz.value
            dev = self.device
            out = CSR(torch.empty(self.n_rows + 1, dtype=torch.int32, device=dev),
                      torch.empty(self.nnz, dtype=torch.int32, device=dev),
                      torch.empty(self.nnz, dtype=torch.float64, device=dev),
                      torch.empty(self.nnz, dtype=torch.float64, device=dev))
            c = _csr_ptrs(out)
            _lib.check("efem_p1_numeric", L.efem_p1_numeric(self._plan, ctypes.byref(c), _stream(stream)))
        return out

    def load(self, fq: torch.Tensor, stream=None) -> torch.Tensor:
        b = torch.empty(self.coords.shape[0], dtype=torch.float64, device=self.device)
        fq = fq.contiguous()
        with torch.cuda.device(self.device):
            _lib.check("efem_p1_load", _lib.load().efem_p1_load(self._plan, _ptr(fq), _ptr(b), _stream(stream)))
        return b


def p1_gradient(coords: torch.Tensor, elems: torch.Tensor, v: torch.Tensor, stream=None) -> torch.Tensor:
    """grad v of a P1 field at every quadrature point: (T, nq, dim)."""
    dim = int(coords.shape[1])
    out = torch.empty((elems.shape[0], quad_size(dim), dim), dtype=torch.float64, device=coords.device)
    m = _mesh_struct(coords, elems)
    with torch.cuda.device(coords.device):
        _lib.check("efem_p1_gradient", _lib.load().efem_p1_gradient(ctypes.byref(m), _ptr(v.contiguous()),
                                                                    _ptr(out), _stream(stream)))
    return out


def dirichlet(A: CSR, mask: torch.Tensor, b: torch.Tensor | None = None, stream=None):
    """Symmetric elimination of the masked DOFs (homogeneous values), in place."""
    c = _csr_ptrs(A)
    m = mask.to(torch.uint8).contiguous()
    with torch.cuda.device(A.row_ptr.device):
        _lib.check("efem_dirichlet", _lib.load().efem_dirichlet(ctypes.byref(c), _ptr(m), _ptr(b),
                                                                _stream(stream)))
    return A
