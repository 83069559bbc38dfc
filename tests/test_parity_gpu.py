"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bit-exact: meshes, DOF tables (dofs2nodes, elems2dofs, signs), CSR pattern.
Values: |gpu - oracle| <= 1e-12 * max_j |oracle[i, j]| per row (north_star).
Full BASELINE sizes: sampled rows against the oracle computed row by row,
plus properties that hold at any size (DOF table validity, de Rham, constant
field interpolation, symmetry).
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as ora
from parity import REL_TOL, assert_csr_parity, assert_row_close
from workloads import CONFIGS, NED0, RT0, counts

pytestmark = pytest.mark.gpu

KINDS = [(2, RT0), (2, NED0), (3, RT0), (3, NED0)]
KIND_IDS = ["rt0_2d", "ne0_2d", "rt0_3d", "ne0_3d"]


@pytest.fixture(scope="module")
def api():
    from paper_1409_4618_b200 import api as a

    assert torch.cuda.is_available()
    return a


def _gpu_mesh(api, dim, n, alpha, seed):
    return api.build_mesh(dim, n, alpha, seed, device="cuda:0")


# ---------------------------------------------------------------------------- meshes
@pytest.mark.parametrize("dim,n,alpha,seed", [(2, 1, 0.0, 0), (2, 7, 0.2, 3), (2, 33, 0.1, 9), (3, 1, 0.0, 0),
                                              (3, 5, 0.15, 4), (3, 17, 0.2, 5)])
def test_mesh_bit_exact_small(api, dim, n, alpha, seed):
    c, e = _gpu_mesh(api, dim, n, alpha, seed)
    rc, re = ora.build_mesh(dim, n, alpha, seed)
    assert np.array_equal(e.cpu().numpy(), re)
    assert c.cpu().numpy().tobytes() == rc.tobytes()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_mesh_bit_exact_configs(api, cfg):
    C = CONFIGS[cfg]
    c, e = _gpu_mesh(api, C["dim"], C["n"], C["alpha"], C["seed"])
    rc, re = ora.build_mesh(C["dim"], C["n"], C["alpha"], C["seed"])
    assert np.array_equal(e.cpu().numpy(), re)
    assert c.cpu().numpy().tobytes() == rc.tobytes()


# ---------------------------------------------------------------------------- DOFs + CSR, small
SMALL = {2: [1, 2, 7, 16, 45], 3: [1, 2, 5, 9]}


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_dofs_and_csr_parity_small(api, dim, element):
    for n in SMALL[dim]:
        alpha = 0.2 if dim == 2 else 0.15
        c, e = _gpu_mesh(api, dim, n, alpha, 100 + n)
        ref = ora.assemble(dim, element, c.cpu().numpy(), e.cpu().numpy())
        asm = api.Assembler(c, e, element)
        d2n, e2d, sg = asm.enumerate_dofs()
        assert np.array_equal(d2n.cpu().numpy(), ref.dofs2nodes), n
        assert np.array_equal(e2d.cpu().numpy(), ref.elems2dofs), n
        assert np.array_equal(sg.cpu().numpy(), ref.signs), n
        csr = asm.assemble()
        assert_csr_parity(csr, ref, what=f"n={n}")


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_csr_parity_permuted_unstructured(api, dim, element):
    """Random node relabelling + random local vertex order: the GPU path must
    not depend on the generator's structure (mixed det signs in 2D too)."""
    rng = np.random.default_rng(dim * 10 + element)
    n = 12 if dim == 2 else 4
    rc, re = ora.build_mesh(dim, n, 0.2 if dim == 2 else 0.15, 77)
    perm = rng.permutation(rc.shape[0])
    inv = np.argsort(perm)
    rc = np.ascontiguousarray(rc[perm])
    re = inv[re].astype(np.int32)
    for t in range(re.shape[0]):
        re[t] = re[t][rng.permutation(dim + 1)]
    re = np.ascontiguousarray(re[rng.permutation(re.shape[0])])
    ref = ora.assemble(dim, element, rc, re)
    c = torch.from_numpy(rc).cuda()
    e = torch.from_numpy(re).cuda()
    asm = api.Assembler(c, e, element)
    d2n, e2d, sg = asm.enumerate_dofs()
    assert np.array_equal(d2n.cpu().numpy(), ref.dofs2nodes)
    assert np.array_equal(e2d.cpu().numpy(), ref.elems2dofs)
    assert np.array_equal(sg.cpu().numpy(), ref.signs)
    assert_csr_parity(asm.assemble(), ref, what="permuted")


@pytest.mark.parametrize("cfg", [1])
def test_config1_full_parity(api, cfg):
    C = CONFIGS[cfg]
    c, e = _gpu_mesh(api, C["dim"], C["n"], C["alpha"], C["seed"])
    ref = ora.assemble(C["dim"], C["element"], c.cpu().numpy(), e.cpu().numpy())
    asm = api.Assembler(c, e, C["element"])
    assert_csr_parity(asm.assemble(), ref, what="cfg1")


@pytest.mark.parametrize("dim,element,n", [(2, NED0, 160), (2, RT0, 700), (3, RT0, 14), (3, RT0, 30), (3, NED0, 12),
                                            (3, NED0, 31)],
                         ids=["ne0_2d_160", "rt0_2d_700", "rt0_3d_14", "rt0_3d_30", "ne0_3d_12", "ne0_3d_31"])
def test_csr_parity_medium(api, dim, element, n):
    """Sizes that span many CTA tiles with a ragged tail, full oracle (the
    larger ones run every persistent warp through several grid-stride
    batches)."""
    c, e = _gpu_mesh(api, dim, n, 0.2 if dim == 2 else 0.15, 5)
    ref = ora.assemble(dim, element, c.cpu().numpy(), e.cpu().numpy(), threads=os.cpu_count() or 1)
    asm = api.Assembler(c, e, element)
    assert_csr_parity(asm.assemble(), ref, what="medium")


# ---------------------------------------------------------------------------- API behaviour
def test_numeric_forms_and_determinism(api):
    c, e = _gpu_mesh(api, 3, 6, 0.15, 8)
    asm = api.Assembler(c, e, NED0)
    full = asm.assemble()
    out = asm.alloc_csr()
    out.col_idx.copy_(full.col_idx)
    out.vals_K.zero_()
    asm.numeric(out, forms=api.MASS)
    asm.check()
    assert torch.equal(out.vals_M, full.vals_M)  # bitwise: fixed summation order
    assert torch.count_nonzero(out.vals_K) == 0
    again = asm.assemble()
    for a, b in ((again.vals_M, full.vals_M), (again.vals_K, full.vals_K), (again.col_idx, full.col_idx)):
        assert torch.equal(a, b)


def test_numeric_before_symbolic_is_an_error(api):
    c, e = _gpu_mesh(api, 2, 3, 0.1, 1)
    asm = api.Assembler(c, e, RT0)
    asm.n_rows, asm.nnz = 1, 1
    with pytest.raises(api._lib.EfemError) as ei:
        asm.numeric(asm.alloc_csr(1, 1))
    assert ei.value.status == -9


def test_degenerate_element_reported(api):
    rc, re = ora.build_mesh(2, 4, 0.0, 0)
    bad = 13
    rc = rc.copy()
    # collapse element 13 onto a line: move its third vertex onto the segment of the first two
    v = re[bad]
    rc[v[2]] = 0.5 * (rc[v[0]] + rc[v[1]])
    asm = api.Assembler(torch.from_numpy(rc).cuda(), torch.from_numpy(re).cuda(), NED0)
    with pytest.raises(api._lib.EfemError) as ei:
        asm.assemble()
    assert ei.value.status == -2
    assert 0 <= ei.value.bad_element <= bad  # another element may share the collapse


def test_invalid_node_id_reported(api):
    rc, re = ora.build_mesh(2, 3, 0.0, 0)
    re = re.copy()
    re[5, 1] = rc.shape[0] + 3
    asm = api.Assembler(torch.from_numpy(rc).cuda(), torch.from_numpy(re).cuda(), RT0)
    with pytest.raises(api._lib.EfemError) as ei:
        asm.assemble()
    assert ei.value.status == -1


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
@pytest.mark.parametrize("bad", [-5, 1 << 30], ids=["negative", "2^30"])
@pytest.mark.parametrize("path", ["sync", "async"])
def test_out_of_range_node_ids_reported(api, dim, element, bad, path):
    """A node id outside [0, n_nodes) is EFEM_EINVAL on every path, never an
    illegal address: the kernels after the enumeration's flag return early."""
    rc, re = ora.build_mesh(dim, 3, 0.1, 0)
    asm = api.Assembler(torch.from_numpy(rc).cuda(), torch.from_numpy(re).cuda(), element)
    good = asm.assemble()
    e = torch.from_numpy(re).cuda()
    e[len(re) // 2, 1] = bad
    asm2 = api.Assembler(torch.from_numpy(rc).cuda(), e, element)
    with pytest.raises(api._lib.EfemError) as ei:
        if path == "sync":
            asm2.assemble()
        else:
            asm2.assemble_async(asm.alloc_csr(good.n_rows, good.nnz))
            asm2.check()
    assert ei.value.status == -1
    torch.cuda.synchronize()  # the context is intact
    assert torch.equal(asm.assemble().col_idx, good.col_idx)


def _bowtie_tets():
    """Two tets sharing only the edge (0, 1): a non-manifold fan (its link is
    two disjoint segments)."""
    c = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, -1, 0], [0, 0, -1]], dtype=np.float64)
    e = np.array([[0, 1, 2, 3], [0, 1, 4, 5]], dtype=np.int32)
    return c, e


def test_nonmanifold_edge_rt0_3d_exact(api):
    """Faces need no link count: RT0 3D assembles the bow-tie exactly."""
    c, e = _bowtie_tets()
    ref = ora.assemble(3, RT0, c, e)
    asm = api.Assembler(torch.from_numpy(c).cuda(), torch.from_numpy(e).cuda(), RT0)
    assert_csr_parity(asm.assemble(), ref, what="bowtie")


def test_nonmanifold_edge_ne0_3d_reported(api):
    """NE0 3D sizes edge rows as 1 + 3t + 2[boundary edge], valid when every
    edge's tets form one fan (cycle or path).  A non-manifold edge must be
    reported (EFEM_EINVAL, "non-conforming"), never assembled wrongly."""
    c, e = _bowtie_tets()
    asm = api.Assembler(torch.from_numpy(c).cuda(), torch.from_numpy(e).cuda(), NED0)
    with pytest.raises(api._lib.EfemError) as ei:
        asm.assemble()
    assert ei.value.status == -1


@pytest.mark.parametrize("dim,element", [(3, NED0), (3, RT0), (2, NED0)])
def test_exact_mode_bowtie_and_regular(api, dim, element):
    """efem_plan_set_exact: the non-manifold bow-tie assembles exactly (NE0
    3D), and exact mode changes nothing on a regular mesh (or other kinds)."""
    if dim == 3:
        c, e = _bowtie_tets()
        asm = api.Assembler(torch.from_numpy(c).cuda(), torch.from_numpy(e).cuda(), element)
        asm.set_exact(True)
        assert_csr_parity(asm.assemble(), ora.assemble(3, element, c, e), what="bowtie exact")
    n = 4 if dim == 3 else 9
    cg, eg = _gpu_mesh(api, dim, n, 0.15, 12)
    asm = api.Assembler(cg, eg, element)
    fast = asm.assemble()
    asm.set_exact(True)
    exact = asm.assemble()
    for x, y in zip((fast.row_ptr, fast.col_idx, fast.vals_M, fast.vals_K),
                    (exact.row_ptr, exact.col_idx, exact.vals_M, exact.vals_K)):
        assert torch.equal(x, y)


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_single_element_and_unused_nodes(api, dim, element):
    rc, re = ora.build_mesh(dim, 2, 0.1, 3)
    one = np.ascontiguousarray(re[len(re) // 2: len(re) // 2 + 1])  # all other nodes unused
    ref = ora.assemble(dim, element, rc, one)
    asm = api.Assembler(torch.from_numpy(rc).cuda(), torch.from_numpy(one).cuda(), element)
    assert_csr_parity(asm.assemble(), ref, what="single")


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_empty_mesh(api, dim, element):
    c = torch.zeros((5, dim), dtype=torch.float64, device="cuda")
    e = torch.zeros((0, dim + 1), dtype=torch.int32, device="cuda")
    asm = api.Assembler(c, e, element)
    csr = asm.assemble()
    assert csr.n_rows == 0 and csr.nnz == 0
    assert csr.row_ptr.cpu().tolist() == [0]


def test_assemble_host_matches_device(api):
    C = CONFIGS[1]
    c, e = _gpu_mesh(api, C["dim"], C["n"], C["alpha"], C["seed"])
    asm = api.Assembler(c, e, C["element"])
    dev = asm.assemble()
    h_c = c.cpu().pin_memory()
    h_e = e.cpu().pin_memory()
    d_out = asm.alloc_csr()
    h_out = api.CSR(*(torch.empty_like(t, device="cpu").pin_memory() for t in
                      (dev.row_ptr, dev.col_idx, dev.vals_M, dev.vals_K)))
    c.zero_()  # the host call must upload the mesh itself
    asm.assemble_host(h_c, h_e, d_out, h_out)
    for a, b in ((h_out.row_ptr, dev.row_ptr), (h_out.col_idx, dev.col_idx), (h_out.vals_M, dev.vals_M),
                 (h_out.vals_K, dev.vals_K)):
        assert torch.equal(a, b.cpu())


# ---------------------------------------------------------------------------- full BASELINE sizes
@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_full_config_oracle_parity(api, cfg):
    """north_star's target: at every BASELINE config, the whole CSR of both
    matrices against the oracle (its row-range form on all host cores,
    bitwise the serial oracle): dofs2nodes, elems2dofs, signs, row_ptr and
    col_idx byte for byte; every row of M and K within 1e-12 of the row's
    max |entry|."""
    C = CONFIGS[cfg]
    dim, el, n = C["dim"], C["element"], C["n"]
    c, e = _gpu_mesh(api, dim, n, C["alpha"], C["seed"])
    asm = api.Assembler(c, e, el)
    d2n, e2d, sg = asm.enumerate_dofs()
    d2n, e2d, sg = d2n.cpu().numpy(), e2d.cpu().numpy(), sg.cpu().numpy()
    csr = asm.assemble()
    got = api.CSR(*(t.cpu() for t in (csr.row_ptr, csr.col_idx, csr.vals_M, csr.vals_K)))
    c_h, e_h = c.cpu().numpy(), e.cpu().numpy()
    del csr, asm, c, e
    torch.cuda.empty_cache()
    ref = ora.assemble(dim, el, c_h, e_h, threads=os.cpu_count() or 1)
    assert np.array_equal(d2n, ref.dofs2nodes)
    assert np.array_equal(e2d, ref.elems2dofs)
    assert np.array_equal(sg, ref.signs)
    del d2n, e2d, sg
    assert_csr_parity(got, ref, what=f"cfg{cfg} full")


def _sample_rows(R, rng, k=160):
    fixed = [0, 1, 2, R // 3, R // 2, R - 3, R - 2, R - 1]
    return np.unique(np.concatenate([fixed, rng.integers(0, R, k)]))


def _spmv(row_ptr, col_idx, vals, x):
    A = torch.sparse_csr_tensor(row_ptr.long(), col_idx.long(), vals, (row_ptr.numel() - 1, x.numel()))
    return (A @ x.unsqueeze(1)).squeeze(1)


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_full_config(api, cfg):
    C = CONFIGS[cfg]
    dim, el, n = C["dim"], C["element"], C["n"]
    c, e = _gpu_mesh(api, dim, n, C["alpha"], C["seed"])
    asm = api.Assembler(c, e, el)
    d2n, e2d, sg = asm.enumerate_dofs()
    csr = asm.assemble()
    N, T, R, nnz = counts(dim, el, n)
    assert (csr.n_rows, csr.nnz) == (R, nnz)

    # DOF table validity => numbering = lexicographic rank (unique answer)
    D = d2n.long()
    key = D[:, 0] * (N + 1) ** (D.shape[1] - 1)
    for cc in range(1, D.shape[1]):
        key = key + D[:, cc] * (N + 1) ** (D.shape[1] - 1 - cc)
    assert bool((key[1:] > key[:-1]).all()), "dofs2nodes not strictly lexicographic"
    assert bool((D[:, 1:] > D[:, :-1]).all())
    assert int(torch.bincount(e2d.flatten().long(), minlength=R).min()) >= 1, "unused DOF"
    E = e.long()
    if D.shape[1] == 2:
        st = [(1, 2), (2, 0), (0, 1)] if dim == 2 else [(0, 1), (0, 2), (0, 3), (1, 2), (2, 3), (3, 1)]
        for k, (s0, s1) in enumerate(st):
            a, b = E[:, s0], E[:, s1]
            row = D[e2d[:, k].long()]
            assert torch.equal(row[:, 0], torch.minimum(a, b)) and torch.equal(row[:, 1], torch.maximum(a, b))
            assert torch.equal(sg[:, k].long(), torch.where(a < b, 1, -1))
    else:
        for k in range(4):
            vs = torch.sort(E[:, [v for v in range(4) if v != 3 - k]], dim=1).values
            assert torch.equal(D[e2d[:, k].long()], vs)

    # pattern validity
    rp = csr.row_ptr.long()
    assert int(rp[0]) == 0 and bool((rp[1:] >= rp[:-1]).all()) and int(rp[-1]) == nnz
    ci = csr.col_idx.long()
    same_row = torch.ones(nnz, dtype=torch.bool, device=ci.device)
    same_row[rp[1:-1]] = False
    assert bool((ci[1:][same_row[1:]] > ci[:-1][same_row[1:]]).all()), "columns not strictly ascending"

    # sampled rows against the oracle, row by row
    rng = np.random.default_rng(cfg)
    rows = _sample_rows(R, rng)
    d2n_h = d2n.cpu().numpy()
    res = ora.rows_by_entity(dim, el, c.cpu().numpy(), e.cpu().numpy(), d2n_h[rows])
    rp_h = csr.row_ptr.cpu().numpy()
    for r, (cols, vm, vk) in zip(rows, res):
        lo, hi = rp_h[r], rp_h[r + 1]
        gcols = csr.col_idx[lo:hi].cpu().numpy()
        ek = d2n_h.shape[1]
        assert np.array_equal(d2n_h[gcols], cols[:, :ek]), f"row {r} pattern"
        sub_ptr = np.array([0, hi - lo])
        assert_row_close(csr.vals_M[lo:hi].cpu().numpy(), vm, sub_ptr, what=f"row {r} M")
        assert_row_close(csr.vals_K[lo:hi].cpu().numpy(), vk, sub_ptr, what=f"row {r} K")

    # invariants at full size (any size): constant-field interpolant and de Rham
    v = torch.tensor([0.3, -1.1, 0.7][:dim], dtype=torch.float64, device=c.device)
    X = c
    if el == NED0:
        cvec = ((X[D[:, 1]] - X[D[:, 0]]) * v).sum(1)
    elif dim == 2:
        t = X[D[:, 1]] - X[D[:, 0]]
        cvec = t[:, 1] * v[0] - t[:, 0] * v[1]
    else:
        nu = torch.linalg.cross(X[D[:, 1]] - X[D[:, 0]], X[D[:, 2]] - X[D[:, 0]])
        cvec = 0.5 * (nu * v).sum(1)
    Mc = _spmv(csr.row_ptr, csr.col_idx, csr.vals_M, cvec)
    energy = float((cvec * Mc).sum())
    assert abs(energy - float((v * v).sum())) < 1e-10 * float((v * v).sum())
    Kc = _spmv(csr.row_ptr, csr.col_idx, csr.vals_K, cvec)
    Kabs = _spmv(csr.row_ptr, csr.col_idx, csr.vals_K.abs(), cvec.abs())
    assert float((Kc.abs() / Kabs.clamp_min(1e-300)).max()) < 1e-10
    if el == NED0:
        phi = torch.rand(N, dtype=torch.float64, device=c.device, generator=torch.Generator(c.device).manual_seed(1))
        g = phi[D[:, 1]] - phi[D[:, 0]]
        Kg = _spmv(csr.row_ptr, csr.col_idx, csr.vals_K, g)
        Kga = _spmv(csr.row_ptr, csr.col_idx, csr.vals_K.abs(), g.abs())
        assert float((Kg.abs() / Kga.clamp_min(1e-300)).max()) < 1e-10

    # symmetry of both matrices (pattern symmetric, values to rounding)
    if cfg in (2, 3):
        for vals in (csr.vals_M, csr.vals_K):
            A = torch.sparse_csr_tensor(rp, ci, vals, (R, R)).to_sparse_coo().coalesce()
            At = A.t().coalesce()
            assert torch.equal(A.indices(), At.indices())
            diff = (A.values() - At.values()).abs().max()
            assert float(diff) <= REL_TOL * float(vals.abs().max())


# ---------------------------------------------------------------------------- f4: the paper's L-shape domain
@pytest.mark.parametrize("m,alpha", [(2, 0.0), (8, 0.2), (34, 0.1)])
def test_lshape_bit_exact(api, m, alpha):
    c, e = api.build_lshape(m, alpha, 5, device="cuda:0")
    rc, re = ora.build_lshape(m, alpha, 5)
    assert np.array_equal(e.cpu().numpy(), re)
    assert c.cpu().numpy().tobytes() == rc.tobytes()


@pytest.mark.parametrize("element", [RT0, NED0], ids=["rt0", "ne0"])
def test_lshape_csr_parity(api, element):
    c, e = api.build_lshape(16, 0.15, 9, device="cuda:0")
    ref = ora.assemble(2, element, c.cpu().numpy(), e.cpu().numpy())
    assert_csr_parity(api.Assembler(c, e, element).assemble(), ref, what="lshape")


# ---------------------------------------------------------------------------- asynchronous one-call assembly
@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_assemble_async_equals_two_phase(api, dim, element):
    """efem_assemble_async (counts stay on the device) gives the same CSR,
    byte for byte, as symbolic + numeric; repeated calls are identical."""
    n = 20 if dim == 2 else 5
    c, e = _gpu_mesh(api, dim, n, 0.2 if dim == 2 else 0.15, 31)
    asm = api.Assembler(c, e, element)
    ref = asm.assemble()
    out = asm.alloc_csr()
    for t in (out.row_ptr, out.col_idx, out.vals_M, out.vals_K):
        t.fill_(-7) if t.dtype == torch.int32 else t.fill_(float("nan"))
    for _ in range(2):
        asm.assemble_async(out)
        asm.check()
        for a, b in zip((ref.row_ptr, ref.col_idx, ref.vals_M, ref.vals_K),
                        (out.row_ptr, out.col_idx, out.vals_M, out.vals_K)):
            assert torch.equal(a, b)


def test_assemble_async_capacity_flagged(api):
    c, e = _gpu_mesh(api, 2, 8, 0.1, 2)
    asm = api.Assembler(c, e, NED0)
    full = asm.assemble()
    small = api.CSR(torch.zeros(full.n_rows + 1, dtype=torch.int32, device="cuda"),
                    torch.zeros(full.nnz - 1, dtype=torch.int32, device="cuda"),
                    torch.zeros(full.nnz - 1, dtype=torch.float64, device="cuda"),
                    torch.zeros(full.nnz - 1, dtype=torch.float64, device="cuda"))
    asm.assemble_async(small)
    with pytest.raises(api._lib.EfemError) as ei:
        asm.check()
    assert ei.value.status == -8  # EFEM_ECAPACITY
    assert int(small.col_idx.abs().sum()) == 0  # nothing written


@pytest.mark.parametrize("element", [RT0, NED0], ids=["rt0_2d", "ne0_2d"])
def test_fan_fill_odd_count_and_unaligned_elems(api, element):
    """The fan fill takes two triangles per thread with 8-byte loads: an odd
    triangle count (the last thread's single triangle) and an element array
    only 4-byte aligned (the scalar-load path) give the oracle's CSR too;
    the triangles of each cell share their smallest vertex (one atomic per
    pair) in the generator's order, and not after a shuffle."""
    rc, re = ora.build_mesh(2, 13, 0.2, 31)
    re = np.ascontiguousarray(re[:-1])  # a boundary triangle removed: T odd
    assert re.shape[0] % 2 == 1
    rng = np.random.default_rng(5)
    for order in (np.arange(re.shape[0]), rng.permutation(re.shape[0])):
        ee = np.ascontiguousarray(re[order])
        ref = ora.assemble(2, element, rc, ee)
        c = torch.from_numpy(rc).cuda()
        for offset in (0, 1):  # int32 elements before the array: 0 or 4 bytes
            buf = torch.zeros(ee.size + 4, dtype=torch.int32, device="cuda")
            e = buf[offset:offset + ee.size].view(ee.shape[0], 3)
            e.copy_(torch.from_numpy(ee))
            assert (e.data_ptr() % 8 == 0) == (offset == 0)
            asm = api.Assembler(c, e, element)
            _, e2d, _ = asm.enumerate_dofs()
            assert np.array_equal(e2d.cpu().numpy(), ref.elems2dofs)
            assert_csr_parity(asm.assemble(), ref, what=f"offset={offset}")
