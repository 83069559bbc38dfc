"""ctypes wrapper around liboracle.so (oracle/efem_oracle.cpp).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this module.  The product
path (paper_1409_4618_b200/) never imports it and shares no code with it.

Every function here only marshals numpy arrays; all arithmetic is in the C++
file, which cites the paper passage each step follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "efem_oracle.cpp")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

RT0, NED0 = 0, 1
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -ffp-contract=off, host only)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", "-pthread", "-o", _LIB_PATH, _SRC]
        )
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        vp = ctypes.c_void_p
        L.ora_mesh_sizes.argtypes = [ctypes.c_int, ctypes.c_int, i64p, i64p]
        L.ora_build_mesh.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint64, vp, vp]
        L.ora_n_local_dofs.argtypes = [ctypes.c_int, ctypes.c_int]
        L.ora_ref_basis.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.ora_quadrature.argtypes = [ctypes.c_int, vp, vp]
        L.ora_local_table.argtypes = [ctypes.c_int, ctypes.c_int, vp]
        L.ora_element.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp]
        L.ora_assemble.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, vp, vp,
                                   ctypes.POINTER(ctypes.c_int)]
        L.ora_assemble.restype = ctypes.c_void_p
        L.ora_assemble_blocked.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, vp, vp,
                                           ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.ora_assemble_blocked.restype = ctypes.c_void_p
        L.ora_result_sizes.argtypes = [vp, i64p, i64p]
        L.ora_result_copy.argtypes = [vp] + [vp] * 7
        L.ora_free.argtypes = [vp]
        L.ora_free.restype = None
        L.ora_lshape_sizes.argtypes = [ctypes.c_int, i64p, i64p]
        L.ora_build_lshape.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_uint64, vp, vp]
        L.ora_quad6.argtypes = [ctypes.c_int, vp, vp]
        L.ora_quad_points.argtypes = [ctypes.c_int, ctypes.c_int64, vp, vp, vp]
        L.ora_load.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, vp, vp, vp, vp,
                               ctypes.c_int64, vp, vp]
        L.ora_norm_l2.argtypes = [ctypes.c_int, ctypes.c_int64, vp, vp, vp, ctypes.c_int, vp, vp]
        L.ora_field_error.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp]
        L.ora_p1_assemble.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, vp, vp, ctypes.POINTER(ctypes.c_int)]
        L.ora_p1_assemble.restype = ctypes.c_void_p
        L.ora_p1_load.argtypes = [ctypes.c_int, ctypes.c_int64, vp, vp, ctypes.c_int64, vp, vp]
        L.ora_p1_grad.argtypes = [ctypes.c_int, ctypes.c_int64, vp, vp, vp, vp]
        L.ora_rows_by_entity.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, vp, vp,
                                         ctypes.c_int64, vp, ctypes.c_int, vp, vp, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def n_local_dofs(dim: int, element: int) -> int:
    return lib().ora_n_local_dofs(dim, element)


def mesh_sizes(dim: int, n: int):
    N, T = ctypes.c_int64(), ctypes.c_int64()
    if lib().ora_mesh_sizes(dim, n, ctypes.byref(N), ctypes.byref(T)) != 0:
        raise ValueError("bad mesh size request")
    return N.value, T.value


def build_mesh(dim: int, n: int, alpha: float, seed: int):
    N, T = mesh_sizes(dim, n)
    coords = np.zeros((N, dim), dtype=np.float64)
    elems = np.zeros((T, dim + 1), dtype=np.int32)
    if lib().ora_build_mesh(dim, n, alpha, seed, _p(coords), _p(elems)) != 0:
        raise ValueError("ora_build_mesh failed")
    return coords, elems


def build_lshape(m: int, alpha: float = 0.0, seed: int = 0):
    N, T = ctypes.c_int64(), ctypes.c_int64()
    if lib().ora_lshape_sizes(m, ctypes.byref(N), ctypes.byref(T)) != 0:
        raise ValueError("bad L-shape size")
    coords = np.zeros((N.value, 2))
    elems = np.zeros((T.value, 3), dtype=np.int32)
    lib().ora_build_lshape(m, alpha, seed, _p(coords), _p(elems))
    return coords, elems


def ref_basis(dim: int, element: int, xh):
    m = n_local_dofs(dim, element)
    xh = np.ascontiguousarray(xh, dtype=np.float64)
    nc = 3 if (dim == 3 and element == NED0) else 1
    val = np.zeros((m, dim))
    dc = np.zeros((m, nc))
    lib().ora_ref_basis(dim, element, _p(xh), _p(val), _p(dc))
    return val, dc


def quadrature(dim: int):
    pts = np.zeros((4, dim))
    w = np.zeros(4)
    nip = lib().ora_quadrature(dim, _p(pts), _p(w))
    return pts[:nip].copy(), w[:nip].copy()


def local_table(dim: int, element: int):
    out = np.zeros(24, dtype=np.int32)
    m = lib().ora_local_table(dim, element, _p(out))
    width = 4 if (dim == 3 and element == RT0) else 2
    return out[: m * width].reshape(m, width).copy()


def element(dim: int, element: int, verts, g):
    m = n_local_dofs(dim, element)
    verts = np.ascontiguousarray(verts, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.int32)
    s = np.zeros(m, dtype=np.int8)
    M = np.zeros((m, m))
    K = np.zeros((m, m))
    st = lib().ora_element(dim, element, _p(verts), _p(g), _p(s), _p(M), _p(K))
    if st != 0:
        raise ValueError(f"ora_element failed ({st})")
    return s, M, K


@dataclass
class Assembly:
    dofs2nodes: np.ndarray
    elems2dofs: np.ndarray
    signs: np.ndarray
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals_M: np.ndarray
    vals_K: np.ndarray

    @property
    def n_dofs(self) -> int:
        return self.row_ptr.shape[0] - 1

    def dense(self):
        R = self.n_dofs
        M = np.zeros((R, R))
        K = np.zeros((R, R))
        rows = np.repeat(np.arange(R), np.diff(self.row_ptr))
        M[rows, self.col_idx] = self.vals_M
        K[rows, self.col_idx] = self.vals_K
        return M, K


def assemble(dim: int, element: int, coords, elems, threads: int = 0, blocks: int = 0) -> Assembly:
    """The whole oracle assembly.  threads = 0: the serial ora_assemble;
    threads >= 1: the row-range form ora_assemble_blocked (bitwise the same
    result) on that many threads, over `blocks` node ranges (default 4 per
    thread)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    st = ctypes.c_int()
    if threads:
        h = lib().ora_assemble_blocked(dim, element, coords.shape[0], elems.shape[0], _p(coords), _p(elems),
                                       threads, blocks or 4 * threads, ctypes.byref(st))
    else:
        h = lib().ora_assemble(dim, element, coords.shape[0], elems.shape[0], _p(coords), _p(elems),
                               ctypes.byref(st))
    if not h:
        raise ValueError(f"ora_assemble failed ({st.value})")
    try:
        R, nnz = ctypes.c_int64(), ctypes.c_int64()
        lib().ora_result_sizes(h, ctypes.byref(R), ctypes.byref(nnz))
        R, nnz = R.value, nnz.value
        m = n_local_dofs(dim, element)
        ek = 3 if (dim == 3 and element == RT0) else 2
        out = Assembly(
            dofs2nodes=np.zeros((R, ek), np.int32),
            elems2dofs=np.zeros((elems.shape[0], m), np.int32),
            signs=np.zeros((elems.shape[0], m), np.int8),
            row_ptr=np.zeros(R + 1, np.int32),
            col_idx=np.zeros(nnz, np.int32),
            vals_M=np.zeros(nnz),
            vals_K=np.zeros(nnz),
        )
        lib().ora_result_copy(h, _p(out.dofs2nodes), _p(out.elems2dofs), _p(out.signs), _p(out.row_ptr),
                              _p(out.col_idx), _p(out.vals_M), _p(out.vals_K))
        return out
    finally:
        lib().ora_free(h)


def rows_by_entity(dim: int, element: int, coords, elems, query, cap: int = 64):
    """Sampled rows keyed by column entity (see ora_rows_by_entity)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    q = np.full((len(query), 3), -1, dtype=np.int32)
    q[:, : np.asarray(query).shape[1]] = query
    nq = q.shape[0]
    count = np.zeros(nq, np.int32)
    cols = np.zeros((nq, cap, 3), np.int32)
    vm = np.zeros((nq, cap))
    vk = np.zeros((nq, cap))
    st = lib().ora_rows_by_entity(dim, element, coords.shape[0], elems.shape[0], _p(coords), _p(elems), nq, _p(q),
                                  cap, _p(count), _p(cols), _p(vm), _p(vk))
    if st != 0:
        raise ValueError(f"ora_rows_by_entity failed ({st})")
    return [(cols[i, : count[i]], vm[i, : count[i]], vk[i, : count[i]]) for i in range(nq)]


# --------------------------------------------------------------------------- f1: vectorized integration
VALUE, DERIVATIVE = 0, 1


def quad6(dim: int):
    """Degree-6 rule on the reference element: points (nq, dim), weights (nq,)."""
    pts = np.zeros((24, dim))
    w = np.zeros(24)
    nq = lib().ora_quad6(dim, _p(pts), _p(w))
    return pts[:nq].copy(), w[:nq].copy()


def quad_points(dim: int, coords, elems):
    """Physical degree-6 quadrature points, shape (T, nq, dim)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    nq = 12 if dim == 2 else 24
    out = np.zeros((elems.shape[0], nq, dim))
    lib().ora_quad_points(dim, elems.shape[0], _p(coords), _p(elems), _p(out))
    return out


def load(dim: int, element: int, pairing: int, coords, elems, asm: Assembly, fq):
    """b_i = sum_K sum_q w |det| f . (phi_i or its div / curl) at the points."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    fq = np.ascontiguousarray(fq, dtype=np.float64)
    b = np.zeros(asm.n_dofs)
    st = lib().ora_load(dim, element, pairing, elems.shape[0], _p(coords), _p(elems),
                        _p(np.ascontiguousarray(asm.elems2dofs)), _p(np.ascontiguousarray(asm.signs)), asm.n_dofs,
                        _p(fq), _p(b))
    if st != 0:
        raise ValueError(f"ora_load failed ({st})")
    return b


def norm_l2(dim: int, coords, elems, fq):
    """(total, per_element) of sum_K sum_q w |det| |f|^2; fq shape (T, nq[, nf])."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    fq = np.ascontiguousarray(fq, dtype=np.float64)
    nf = 1 if fq.ndim == 2 else fq.shape[2]
    per = np.zeros(elems.shape[0])
    tot = ctypes.c_double()
    lib().ora_norm_l2(dim, elems.shape[0], _p(coords), _p(elems), _p(fq), nf, _p(per), ctypes.byref(tot))
    return tot.value, per


def field_error(dim: int, element: int, coords, elems, asm: Assembly, coeffs, Eq, Dq):
    """(||E - v||^2, ||D E - D v||^2) for v = sum_i coeffs_i phi_i, D = div / curl."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    err = np.zeros(2)
    st = lib().ora_field_error(dim, element, elems.shape[0], _p(coords), _p(elems),
                               _p(np.ascontiguousarray(asm.elems2dofs)), _p(np.ascontiguousarray(asm.signs)),
                               _p(np.ascontiguousarray(coeffs, dtype=np.float64)),
                               _p(np.ascontiguousarray(Eq, dtype=np.float64)),
                               _p(np.ascontiguousarray(Dq, dtype=np.float64)), _p(err))
    if st != 0:
        raise ValueError(f"ora_field_error failed ({st})")
    return err[0], err[1]


# --------------------------------------------------------------------------- f3: P1 (for the majorant example)
def p1_assemble(dim: int, coords, elems):
    """P1 (nodal) CSR over the nodes: (row_ptr, col_idx, vals_M, vals_K)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    st = ctypes.c_int()
    h = lib().ora_p1_assemble(dim, coords.shape[0], elems.shape[0], _p(coords), _p(elems), ctypes.byref(st))
    if not h:
        raise ValueError(f"ora_p1_assemble failed ({st.value})")
    try:
        R, nnz = ctypes.c_int64(), ctypes.c_int64()
        lib().ora_result_sizes(h, ctypes.byref(R), ctypes.byref(nnz))
        rp = np.zeros(R.value + 1, np.int32)
        ci = np.zeros(nnz.value, np.int32)
        vm = np.zeros(nnz.value)
        vk = np.zeros(nnz.value)
        lib().ora_result_copy(h, None, None, None, _p(rp), _p(ci), _p(vm), _p(vk))
        return rp, ci, vm, vk
    finally:
        lib().ora_free(h)


def p1_load(dim: int, coords, elems, fq):
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    b = np.zeros(coords.shape[0])
    lib().ora_p1_load(dim, elems.shape[0], _p(coords), _p(elems), coords.shape[0],
                      _p(np.ascontiguousarray(fq, dtype=np.float64)), _p(b))
    return b


def p1_grad(dim: int, coords, elems, v):
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    elems = np.ascontiguousarray(elems, dtype=np.int32)
    g = np.zeros((elems.shape[0], dim))
    lib().ora_p1_grad(dim, elems.shape[0], _p(coords), _p(elems), _p(np.ascontiguousarray(v, dtype=np.float64)),
                      _p(g))
    return g
