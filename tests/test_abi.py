"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/efem.h declares, and rejects bad arguments before touching CUDA."""
import ctypes

import pytest

from paper_1409_4618_b200 import _lib


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    names = _lib.declared_symbols()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n


def test_status_strings():
    L = _lib.load()
    for code, name in [(0, "EFEM_OK"), (-1, "EFEM_EINVAL"), (-2, "EFEM_EDEGENERATE"), (-5, "EFEM_EOVERFLOW"),
                       (-8, "EFEM_ECAPACITY"), (-9, "EFEM_ESTATE")]:
        assert L.efem_status_string(code).decode() == name


@pytest.mark.parametrize("dim,n,N,T", [(2, 1, 4, 2), (2, 16, 289, 512), (3, 1, 8, 6), (3, 128, 2146689, 12582912),
                                       (2, 4096, 16785409, 33554432)])
def test_mesh_sizes(dim, n, N, T):
    L = _lib.load()
    a, b = ctypes.c_int64(), ctypes.c_int64()
    assert L.efem_mesh_sizes(dim, n, ctypes.byref(a), ctypes.byref(b)) == 0
    assert (a.value, b.value) == (N, T)


def test_mesh_sizes_rejects():
    L = _lib.load()
    a, b = ctypes.c_int64(), ctypes.c_int64()
    assert L.efem_mesh_sizes(4, 2, ctypes.byref(a), ctypes.byref(b)) == -1
    assert L.efem_mesh_sizes(2, 0, ctypes.byref(a), ctypes.byref(b)) == -1
    assert L.efem_mesh_sizes(3, 1000, ctypes.byref(a), ctypes.byref(b)) == -5  # 6e9 tets: int32 overflow


def test_build_mesh_rejects_bad_jitter_before_cuda():
    L = _lib.load()
    # 2D limit 1/(2 sqrt(4)) = 0.25
    assert L.efem_build_mesh(2, 4, 0.25, 0, ctypes.c_void_p(16), ctypes.c_void_p(16), None) == -1
    assert L.efem_build_mesh(2, 4, -0.1, 0, ctypes.c_void_p(16), ctypes.c_void_p(16), None) == -1
    assert L.efem_build_mesh(2, 4, 0.1, 0, None, ctypes.c_void_p(16), None) == -1


def test_plan_create_rejects_bad_mesh_before_cuda():
    L = _lib.load()
    plan = ctypes.c_void_p()
    ws = ctypes.c_size_t()
    bad_dim = _lib.efem_mesh(4, 10, 10, 16, 16)
    assert L.efem_plan_create(ctypes.byref(plan), ctypes.byref(bad_dim), 0, ctypes.byref(ws)) == -1
    m = _lib.efem_mesh(2, 10, 10, 16, 16)
    assert L.efem_plan_create(ctypes.byref(plan), ctypes.byref(m), 7, ctypes.byref(ws)) == -1
    misaligned = _lib.efem_mesh(3, 10, 10, 16, 20)
    assert L.efem_plan_create(ctypes.byref(plan), ctypes.byref(misaligned), 1, ctypes.byref(ws)) == -1
    huge = _lib.efem_mesh(3, 10, 1 << 28, 16, 16)
    assert L.efem_plan_create(ctypes.byref(plan), ctypes.byref(huge), 1, ctypes.byref(ws)) == -5
    assert L.efem_plan_create(None, ctypes.byref(m), 0, ctypes.byref(ws)) == -1
