"""Comparison helpers for GPU-vs-oracle parity (tolerances from BASELINE.json
north_star: bit-exact pattern and DOF numbering; values within 1e-12 of each
row's max |entry|, fp64)."""
import numpy as np

REL_TOL = 1e-12


def assert_row_close(got, want, row_ptr, tol=REL_TOL, what=""):
    """|got - want| <= tol * max_j |want[i, j]| for every row i."""
    got = np.asarray(got)
    want = np.asarray(want)
    if want.size == 0:
        assert got.size == 0
        return
    starts = row_ptr[:-1]
    nz = np.diff(row_ptr) > 0
    scale = np.zeros(len(starts))
    scale[nz] = np.maximum.reduceat(np.abs(want), starts[nz])
    rows = np.repeat(np.arange(len(starts)), np.diff(row_ptr))
    err = np.abs(got - want)
    bad = err > tol * scale[rows]
    if bad.any():
        i = int(np.argmax(err / np.maximum(scale[rows], 1e-300)))
        raise AssertionError(f"{what}: {int(bad.sum())} entries off; worst at {i}: got {got[i]!r} want {want[i]!r} "
                             f"row scale {scale[rows][i]!r}")


def assert_csr_parity(gpu_csr, ref, what=""):
    row_ptr = gpu_csr.row_ptr.cpu().numpy()
    col_idx = gpu_csr.col_idx.cpu().numpy()
    assert np.array_equal(row_ptr, ref.row_ptr), f"{what}: row_ptr differs"
    assert np.array_equal(col_idx, ref.col_idx), f"{what}: col_idx differs"
    assert_row_close(gpu_csr.vals_M.cpu().numpy(), ref.vals_M, ref.row_ptr, what=what + " M")
    assert_row_close(gpu_csr.vals_K.cpu().numpy(), ref.vals_K, ref.row_ptr, what=what + " K")
