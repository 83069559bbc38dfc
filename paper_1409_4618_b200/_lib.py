"""ctypes binding of libefem.so (include/efem.h).  Argument marshalling only.

Loads the in-tree ``libefem.so``; there is no fallback of any kind: if the
library is missing the import fails loudly (build it with
``python -m paper_1409_4618_b200.build`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libefem.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "efem.h")

EFEM_OK = 0
EFEM_RT0, EFEM_NED0 = 0, 1
EFEM_MASS, EFEM_STIFF, EFEM_PATTERN, EFEM_ALL = 1, 2, 4, 7
EFEM_PAIR_VALUE, EFEM_PAIR_DERIV = 0, 1


class efem_mesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n_nodes", ctypes.c_int64), ("n_elems", ctypes.c_int64),
                ("coords", ctypes.c_void_p), ("elems", ctypes.c_void_p)]


class efem_dofs(ctypes.Structure):
    _fields_ = [("n_dofs", ctypes.c_int64), ("dofs2nodes", ctypes.c_void_p), ("elems2dofs", ctypes.c_void_p),
                ("signs", ctypes.c_void_p)]


class efem_csr(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col_idx", ctypes.c_void_p), ("vals_mass", ctypes.c_void_p), ("vals_stiff", ctypes.c_void_p)]


class EfemError(RuntimeError):
    def __init__(self, fn, status, lib):
        self.status = status
        name = lib.efem_status_string(status).decode()
        msg = lib.efem_last_error().decode()
        self.bad_element = lib.efem_last_bad_element() if name == "EFEM_EDEGENERATE" else -1
        super().__init__(f"{fn}: {name} ({status}): {msg}")


_lib = None


def declared_symbols():
    """Function names declared in include/efem.h."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(efem_[a-z_0-9]+)\s*\(", src)))


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libefem.so not built at {LIB_PATH}; run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i64p = ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)
    st = ctypes.c_int
    sig = {
        "efem_mesh_sizes": (st, [ctypes.c_int, ctypes.c_int, i64p, i64p]),
        "efem_build_mesh": (st, [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint64, vp, vp, vp]),
        "efem_plan_create": (st, [ctypes.POINTER(vp), ctypes.POINTER(efem_mesh), ctypes.c_int,
                                  ctypes.POINTER(ctypes.c_size_t)]),
        "efem_plan_set_workspace": (st, [vp, vp, ctypes.c_size_t]),
        "efem_plan_destroy": (st, [vp]),
        "efem_plan_set_exact": (st, [vp, ctypes.c_int]),
        "efem_enumerate_dofs": (st, [vp, ctypes.POINTER(efem_dofs), vp]),
        "efem_assemble_symbolic": (st, [vp, i64p, i64p, vp, vp]),
        "efem_assemble_numeric": (st, [vp, ctypes.c_uint, ctypes.POINTER(efem_csr), vp]),
        "efem_plan_check": (st, [vp, vp]),
        "efem_plan_check_async": (st, [vp, vp]),
        "efem_assemble_async": (st, [vp, ctypes.c_uint, ctypes.POINTER(efem_csr), vp]),
        "efem_assemble_host": (st, [vp, vp, vp, ctypes.POINTER(efem_csr), ctypes.POINTER(efem_csr), vp]),
        "efem_partition": (st, [ctypes.POINTER(efem_mesh), i64, i64, vp, ctypes.POINTER(ctypes.c_size_t), i64p, i64p, vp, vp, vp, vp]),
        "efem_part_counts": (st, [vp, vp, i64, i64, vp, i64p, vp]),
        "efem_part_scan": (st, [vp, i64, vp, vp, ctypes.POINTER(ctypes.c_size_t), vp]),
        "efem_part_globalize": (st, [vp, vp, vp, vp, vp]),
        "efem_part_numeric": (st, [vp, ctypes.c_uint, i64p, i64, vp, ctypes.POINTER(efem_csr), vp]),
        "efem_part_bind": (st, [vp, vp, i64, i64, vp]),
        "efem_part_enumerate_async": (st, [vp, vp, vp]),
        "efem_part_numeric_async": (st, [vp, ctypes.c_uint, vp, ctypes.POINTER(efem_csr), vp]),
        "efem_part_window": (st, [vp, vp, vp]),
        "efem_lshape_sizes": (st, [ctypes.c_int, i64p, i64p]),
        "efem_build_mesh_lshape": (st, [ctypes.c_int, ctypes.c_double, ctypes.c_uint64, vp, vp, vp]),
        "efem_quad_size": (ctypes.c_int, [ctypes.c_int]),
        "efem_quad_points": (st, [ctypes.POINTER(efem_mesh), vp, vp]),
        "efem_assemble_load": (st, [vp, ctypes.c_int, vp, vp, vp]),
        "efem_norm_l2": (st, [ctypes.POINTER(efem_mesh), vp, ctypes.c_int, vp, vp, vp,
                              ctypes.POINTER(ctypes.c_size_t), vp]),
        "efem_field_error": (st, [vp, vp, vp, vp, vp, vp, ctypes.POINTER(ctypes.c_size_t), vp]),
        "efem_spmv": (st, [ctypes.POINTER(efem_csr), ctypes.c_double, ctypes.c_double, vp, vp, vp]),
        "efem_cg": (st, [ctypes.POINTER(efem_csr), ctypes.c_double, ctypes.c_double, vp, vp, ctypes.c_double,
                         ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), vp,
                         ctypes.POINTER(ctypes.c_size_t), vp]),
        "efem_p1_plan_create": (st, [ctypes.POINTER(vp), ctypes.POINTER(efem_mesh), ctypes.POINTER(ctypes.c_size_t)]),
        "efem_p1_plan_set_workspace": (st, [vp, vp, ctypes.c_size_t]),
        "efem_p1_plan_destroy": (st, [vp]),
        "efem_p1_symbolic": (st, [vp, i64p, i64p, vp]),
        "efem_p1_numeric": (st, [vp, ctypes.POINTER(efem_csr), vp]),
        "efem_p1_load": (st, [vp, vp, vp, vp]),
        "efem_p1_gradient": (st, [ctypes.POINTER(efem_mesh), vp, vp, vp]),
        "efem_dirichlet": (st, [ctypes.POINTER(efem_csr), vp, vp, vp]),
        "efem_part_add_offset": (st, [vp, i64, vp, ctypes.c_int, vp]),
        "efem_index_gather": (st, [vp, vp, vp, i64, ctypes.c_int32, vp]),
        "efem_index_scatter": (st, [vp, vp, vp, i64, vp]),
        "efem_part_globalize_sub": (st, [vp, vp, i64, i64, vp, vp]),
        "efem_comm_unique_id": (st, [vp]),
        "efem_comm_init": (st, [ctypes.POINTER(vp), vp, ctypes.c_int, ctypes.c_int]),
        "efem_comm_destroy": (st, [vp]),
        "efem_dist_plan_create": (st, [ctypes.POINTER(vp), ctypes.POINTER(efem_mesh), ctypes.c_int, i64, i64, vp, vp]),
        "efem_dist_group_create": (st, [vp, ctypes.c_int, ctypes.POINTER(efem_mesh), ctypes.c_int, vp, vp]),
        "efem_dist_layout": (st, [vp, i64, i64, vp, ctypes.c_int, ctypes.c_int, vp]),
        "efem_dist_info": (st, [vp, vp]),
        "efem_dist_assemble": (st, [vp, ctypes.c_uint, ctypes.POINTER(efem_csr), vp]),
        "efem_dist_assemble_group": (st, [vp, ctypes.c_int, ctypes.c_uint, vp, vp]),
        "efem_dist_check": (st, [vp, vp, vp]),
        "efem_dist_plan_destroy": (st, [vp]),
        "efem_status_string": (ctypes.c_char_p, [st]),
        "efem_last_error": (ctypes.c_char_p, []),
        "efem_last_bad_element": (i64, []),
        "efem_launch_count": (i64, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(fn: str, status: int):
    if status != EFEM_OK:
        raise EfemError(fn, status, load())
