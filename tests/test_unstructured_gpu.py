"""GPU parity on genuinely unstructured meshes (scipy Delaunay of seeded
random points) and on high-valence fans: irregular valences drive the
enumeration's fallbacks (2D buckets of > 8 instances, 3D nodes with more
larger neighbours / faces than the register lists hold) and the NE0-3D
rows with more than 7 tets (row_generic).  Bit-exact DOF tables and pattern,
values within 1e-12 of each row's max, as everywhere else."""
import numpy as np
import pytest
import torch
from scipy.spatial import Delaunay

from oracle import oracle as ora
from parity import REL_TOL
from workloads import NED0, RT0

pytestmark = pytest.mark.gpu

KINDS = [(2, RT0), (2, NED0), (3, RT0), (3, NED0)]
KIND_IDS = ["rt0_2d", "ne0_2d", "rt0_3d", "ne0_3d"]


def delaunay_mesh(dim, n_pts, seed):
    """Delaunay mesh of n_pts seeded random points in the unit square / cube
    (corners included), non-flat elements only."""
    rng = np.random.default_rng(seed)
    corners = np.array(np.meshgrid(*[[0.0, 1.0]] * dim, indexing="ij")).reshape(dim, -1).T
    pts = np.concatenate([corners, rng.random((n_pts, dim))])
    el = Delaunay(pts).simplices.astype(np.int32)
    el = el[quality(pts, el) > 1e-12]
    used = np.unique(el)  # drop points no element references (qhull may skip coplanar ones)
    remap = -np.ones(pts.shape[0], np.int64)
    remap[used] = np.arange(used.size)
    return np.ascontiguousarray(pts[used]), np.ascontiguousarray(remap[el].astype(np.int32))


def quality(pts, el):
    """|det B_K| / (longest edge)^d: ~0.1-0.4 for well-shaped elements, -> 0
    for slivers (whose local matrices are ill-conditioned: two different fp64
    evaluations of the same integral then differ by ~eps / quality^2)."""
    x = pts[el]
    d = x.shape[1] - 1
    vol = np.abs(np.linalg.det(x[:, 1:] - x[:, :1]))
    L = np.max(np.stack([np.linalg.norm(x[:, i] - x[:, j], axis=1) for i in range(d + 1)
                         for j in range(i + 1, d + 1)]), axis=0)
    return vol / L ** d


def fan_mesh(k, seed):
    """Node 0 at the centre of k triangles (0, i, i+1) closing a disc: node 0
    owns 2k edge instances (2D bucket fallback); ids shuffled except the centre."""
    rng = np.random.default_rng(seed)
    ang = np.sort(rng.random(k)) * 2 * np.pi
    r = 0.5 + 0.3 * rng.random(k)
    pts = np.concatenate([[[0.0, 0.0]], np.stack([r * np.cos(ang), r * np.sin(ang)], 1)])
    el = np.array([[0, 1 + i, 1 + (i + 1) % k] for i in range(k)], np.int32)
    perm = np.concatenate([[0], 1 + rng.permutation(k)])
    inv = np.argsort(perm)
    return np.ascontiguousarray(pts[perm]), np.ascontiguousarray(inv[el].astype(np.int32))


# NE0 3D values are compared on rows whose tets all have quality >= Q_MIN:
# the curl-curl entries 4|K|(G_ap G_bq - G_aq G_bp) cancel like 1 / quality^2
# on a sliver, so ANY two fp64 evaluation orders differ there by more than
# 1e-12 of the row max (measured: 1e-8 at quality 3e-5); only those rows'
# pattern is compared.  RT0 (K = s s / |K|) and the 2D forms carry no such
# cancellation and are compared on every row.
Q_MIN = 0.02


def _check(dim, element, pts, el, what, exact=False):
    """Bit-exact DOF tables and pattern everywhere; values within 1e-12 of the
    row max (NE0 3D: on rows of well-shaped tets, see Q_MIN)."""
    from paper_1409_4618_b200 import api

    ref = ora.assemble(dim, element, pts, el)
    asm = api.Assembler(torch.from_numpy(pts).cuda(), torch.from_numpy(el).cuda(), element)
    if exact:
        asm.set_exact(True)
    d2n, e2d, sg = asm.enumerate_dofs()
    assert np.array_equal(d2n.cpu().numpy(), ref.dofs2nodes), what
    assert np.array_equal(e2d.cpu().numpy(), ref.elems2dofs), what
    assert np.array_equal(sg.cpu().numpy(), ref.signs), what
    bad_dof = np.zeros(ref.n_dofs, bool)
    if dim == 3 and element == NED0:
        bad_dof[ref.elems2dofs[quality(pts, el) < Q_MIN].ravel()] = True
    rows = np.repeat(np.arange(ref.n_dofs), np.diff(ref.row_ptr))
    good = ~bad_dof[rows]
    assert good.mean() > 0.5, what  # most of the matrix is compared
    out_sync = asm.assemble()
    out_async = asm.alloc_csr()
    asm.assemble_async(out_async, api.ALL)
    asm.check()
    for out, tag in ((out_sync, ""), (out_async, " async")):
        assert np.array_equal(out.row_ptr.cpu().numpy(), ref.row_ptr), what + tag
        assert np.array_equal(out.col_idx.cpu().numpy(), ref.col_idx), what + tag
        for got, want, f in ((out.vals_M, ref.vals_M, "M"), (out.vals_K, ref.vals_K, "K")):
            got = got.cpu().numpy()
            scale = np.zeros(ref.n_dofs)
            nz = np.diff(ref.row_ptr) > 0
            scale[nz] = np.maximum.reduceat(np.abs(want), ref.row_ptr[:-1][nz])
            err = np.abs(got - want)[good]
            assert (err <= REL_TOL * scale[rows][good]).all(), (what + tag + " " + f,
                                                                 float((err / scale[rows][good]).max()))
    return ref


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
@pytest.mark.parametrize("seed", [1, 2])
def test_delaunay_parity(dim, element, seed):
    pts, el = delaunay_mesh(dim, 3000 if dim == 2 else 700, seed)
    ref = _check(dim, element, pts, el, f"delaunay{dim}d seed {seed}")
    if dim == 3 and element == NED0:
        # the mesh must actually exercise the > 7-tets-per-edge rows
        t = np.zeros(ref.n_dofs, np.int64)
        np.add.at(t, ref.elems2dofs.ravel(), 1)
        assert t.max() > 7


def test_delaunay_filtered_nonmanifold_exact_mode():
    """Slivers removed (quality >= Q_MIN everywhere): the holes leave edges
    whose tets form several fans (non-manifold), which the default closed-form
    row sizing flags and exact mode (efem_plan_set_exact) sizes by counting
    link vertices.  Exact mode must match the oracle on every row."""
    pts, el = delaunay_mesh(3, 700, 1)
    el = np.ascontiguousarray(el[quality(pts, el) >= Q_MIN])
    _check(3, NED0, pts, el, "filtered delaunay exact", exact=True)
    _check(3, RT0, pts, el, "filtered delaunay rt0")


@pytest.mark.parametrize("element", [RT0, NED0], ids=["rt0", "ne0"])
@pytest.mark.parametrize("k", [5, 40, 200])
def test_fan_parity(element, k):
    pts, el = fan_mesh(k, k)
    _check(2, element, pts, el, f"fan k={k}")


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_delaunay_sweep_small(dim, element):
    """Many tiny unstructured meshes (4 .. 60 random points, 12 seeds): one to
    a few hundred elements, mostly boundary entities -- DOF tables, pattern
    and values against the oracle, both assembly paths."""
    for seed in range(12):
        n_pts = [1, 2, 5, 9, 17, 30, 45, 60][seed % 8]
        pts, el = delaunay_mesh(dim, n_pts, 100 + seed)
        if el.shape[0] == 0:
            continue
        _check(dim, element, pts, el, f"sweep {dim}d n={n_pts} seed={seed}")


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
@pytest.mark.parametrize("P", [3, 5])
def test_delaunay_partitioned_async(dim, element, P):
    """Row-owned partitions of an unstructured mesh (irregular sub-meshes,
    uneven ownership), asynchronous form: the slices concatenate to the
    1-GPU CSR byte for byte."""
    from paper_1409_4618_b200 import api, dist

    pts, el = delaunay_mesh(dim, 1500 if dim == 2 else 300, 7)
    coords, elems = torch.from_numpy(pts).cuda(), torch.from_numpy(el).cuda()
    one = api.Assembler(coords, elems, element).assemble()
    from test_dist_gpu import _exchange, _parts

    ranges, parts = _parts(coords, elems, element, P)
    W = max(hi - lo for lo, hi in ranges)
    _exchange(parts, [p.symbolic() for p in parts])
    caps = [p.alloc_slice() for p in parts]
    for p in parts:
        p.bind(W, P)
    _exchange(parts, [p.enumerate_async() for p in parts])
    for p, c in zip(parts, caps):
        p.numeric_async(c)
        p.check()
    offs, total = dist.offsets_from_counts([int(p.window[3].item()) for p in parts])
    assert total == one.nnz
    rp, ci, vm, vk = dist.concat_slices(caps, offs)
    assert np.array_equal(rp, one.row_ptr.cpu().numpy()) and np.array_equal(ci, one.col_idx.cpu().numpy())
    assert np.array_equal(vm, one.vals_M.cpu().numpy()) and np.array_equal(vk, one.vals_K.cpu().numpy())


@pytest.mark.parametrize("dim,element", [(3, NED0), (2, NED0)], ids=["ne0_3d", "ne0_2d"])
def test_node_ids_beyond_2e27(dim, element):
    """Node ids straddling 2^27 (a coordinate array of 2^27 + 64 nodes, most of
    them unused): the NE0-3D fast path packs node ids into 27 bits and must
    hand such meshes to the generic path.  The relabelling is monotone, so
    DOF numbering, signs and values equal the compact mesh's (oracle)."""
    from paper_1409_4618_b200 import api

    pts, el = delaunay_mesh(dim, 40 if dim == 3 else 60, 3)
    ref = ora.assemble(dim, element, pts, el)
    n = pts.shape[0]
    off = (1 << 27) - n // 2
    N = off + n
    coords = torch.zeros((N, dim), dtype=torch.float64, device="cuda")
    coords[off:] = torch.from_numpy(pts).cuda()
    elems = torch.from_numpy(el + off).cuda()
    asm = api.Assembler(coords, elems, element)
    out = asm.assemble()
    assert np.array_equal(out.row_ptr.cpu().numpy(), ref.row_ptr)
    assert np.array_equal(out.col_idx.cpu().numpy(), ref.col_idx)
    for got, want in ((out.vals_M, ref.vals_M), (out.vals_K, ref.vals_K)):
        got = got.cpu().numpy()
        scale = np.maximum.reduceat(np.abs(want), ref.row_ptr[:-1])
        rows = np.repeat(np.arange(ref.n_dofs), np.diff(ref.row_ptr))
        if dim == 3:  # (see Q_MIN: rows of slivers are conditioning-limited)
            bad = np.zeros(ref.n_dofs, bool)
            bad[ref.elems2dofs[quality(pts, el) < Q_MIN].ravel()] = True
            keep = ~bad[rows]
        else:
            keep = np.ones(rows.size, bool)
        assert (np.abs(got - want)[keep] <= REL_TOL * scale[rows][keep]).all()
    del asm, out, coords
    torch.cuda.empty_cache()


def test_ne3_sliver_rows_against_exact_rationals():
    """The NE0-3D rows that _check leaves out of the 1e-12 value comparison
    (rows touching tets of quality < Q_MIN) are checked against the EXACT
    matrix entries: the fp64 coordinates are exact rationals, so
    bruteforce.element_matrices(exact=True) (physical-space DOF duality in
    fractions.Fraction, no Piola, no quadrature) gives the exact local
    matrices of PAPER.md:352-363.  Both fp64 evaluations (the GPU's closed
    form and the oracle's quadrature) must sit within the conditioning bound
    16 eps / q^2 of the row max (q = the smallest quality among the row's
    tets: the curl-curl entries cancel like 1 / q^2); the GPU is not allowed
    to be the worse one by more than that bound either."""
    import bruteforce
    from paper_1409_4618_b200 import api

    pts, el = delaunay_mesh(3, 700, 1)
    q = quality(pts, el)
    ref = ora.assemble(3, NED0, pts, el)
    asm = api.Assembler(torch.from_numpy(pts).cuda(), torch.from_numpy(el).cuda(), NED0)
    out = asm.assemble()
    gm, gk = out.vals_M.cpu().numpy(), out.vals_K.cpu().numpy()
    rp, ci = ref.row_ptr, ref.col_idx
    # rows of the worst slivers
    qmin_row = np.full(ref.n_dofs, np.inf)
    np.minimum.at(qmin_row, ref.elems2dofs.ravel(), np.repeat(q, 6))
    rows = np.argsort(qmin_row)[:24]
    assert qmin_row[rows].max() < Q_MIN
    tets_of = {}
    for t in range(el.shape[0]):
        for k in range(6):
            tets_of.setdefault(int(ref.elems2dofs[t, k]), []).append(t)
    d2n = [tuple(r) for r in ref.dofs2nodes]
    eps = np.finfo(float).eps
    worst = 0.0
    for r in rows:
        exact_m, exact_k = {}, {}
        for t in tets_of[int(r)]:
            g = [int(v) for v in el[t]]
            keys, M, K = bruteforce.element_matrices(3, NED0, pts[g].tolist(), g, exact=True)
            kr = keys.index(d2n[r])
            for l, key in enumerate(keys):
                exact_m[key] = exact_m.get(key, 0) + M[kr][l]
                exact_k[key] = exact_k.get(key, 0) + K[kr][l]
        lo, hi = rp[r], rp[r + 1]
        cols = [d2n[c] for c in ci[lo:hi]]
        assert sorted(cols) == sorted(exact_m)  # the pattern is the exact one
        bound = 16 * eps / qmin_row[r] ** 2
        for got, ora_v, ex in ((gm, ref.vals_M, exact_m), (gk, ref.vals_K, exact_k)):
            xv = np.array([float(ex[c]) for c in cols])
            scale = np.abs(xv).max()
            e_gpu = np.abs(got[lo:hi] - xv).max() / scale
            e_ora = np.abs(ora_v[lo:hi] - xv).max() / scale
            assert e_gpu <= bound, (int(r), e_gpu, e_ora, bound)
            assert e_ora <= bound, (int(r), e_gpu, e_ora, bound)
            worst = max(worst, e_gpu * qmin_row[r] ** 2 / eps)
    print(f"worst GPU error x q^2 / eps over the sliver rows: {worst:.3g}")


def _max_fan(el, n_nodes):
    """Largest node fan of the 2D fan pipeline: triangles in which the node
    is the smallest or the middle vertex."""
    s = np.sort(el, axis=1)
    return int(np.bincount(s[:, :2].ravel(), minlength=n_nodes).max())


@pytest.mark.parametrize("element", [RT0, NED0], ids=["rt0_2d", "ne0_2d"])
def test_fan_register_path_choice_on_swapped_mesh(element):
    """The fan pass launches its 4-triangle register kernel when the plan's
    previous pass saw no larger fan (fan2d.cu FAN_SMALL).  Swap a relabelled
    copy of the mesh (same sizes, fans of up to 6+ triangles) into the plan's
    buffers: the 4-kernel's slow path for the big fans, the synchronous and
    the graph-replayed asynchronous path, and the next call (back on the
    8-kernel) must all give the CSR of a fresh plan, bit for bit."""
    from paper_1409_4618_b200 import api
    coords, elems = api.build_mesh(2, 48, 0.2, 11)
    n_nodes = coords.shape[0]
    el1 = elems.cpu().numpy()
    assert _max_fan(el1, n_nodes) <= 4
    rng = np.random.default_rng(5)
    perm = rng.permutation(n_nodes)  # new id of node i: perm[i]
    c2 = torch.empty_like(coords)
    c2[torch.from_numpy(perm).to(coords.device)] = coords
    e2 = torch.from_numpy(perm[el1].astype(np.int32)).to(elems.device)
    assert _max_fan(e2.cpu().numpy(), n_nodes) > 4

    ref = api.Assembler(c2.clone(), e2.clone(), element).assemble()

    asm = api.Assembler(coords, elems, element)
    asm.symbolic()                      # structured mesh: the next fan pass takes the 4-kernel
    out = asm.alloc_csr()
    asm.assemble_async(out, api.ALL)    # graph captured with the 4-kernel
    asm.check()
    asm.coords.copy_(c2)
    asm.elems.copy_(e2)
    outs = []
    asm.symbolic()                      # synchronous, 4-kernel, on the swapped mesh
    o = asm.alloc_csr()
    asm.numeric(o, api.ALL)
    asm.check()
    outs.append(o)
    asm.assemble_async(out, api.ALL)    # replay of the 4-kernel graph on the swapped mesh
    asm.check()
    outs.append(_csr_copy(out))
    asm.symbolic()                      # the 8-kernel (this mesh's fans were seen)
    o = asm.alloc_csr()
    asm.numeric(o, api.ALL)
    asm.check()
    outs.append(o)
    for o in outs:
        for a, b in ((o.row_ptr, ref.row_ptr), (o.col_idx, ref.col_idx), (o.vals_M, ref.vals_M),
                     (o.vals_K, ref.vals_K)):
            assert torch.equal(a, b)


def _csr_copy(c):
    from paper_1409_4618_b200 import api
    return api.CSR(c.row_ptr.clone(), c.col_idx.clone(), c.vals_M.clone(), c.vals_K.clone())


def edge_ring_mesh(k, rings=1):
    """rings x k tets (0, p, r_i, r_(i+1) mod k) around the edges (0, p), p the
    pole of each ring (ring 1 above node 0, ring 2 below): node 0 is the
    smallest vertex of all of them (its fan in the NE0-3D enumeration), with
    rings * (k + 1) distinct larger neighbours, and each edge (0, p) has k tets."""
    pts, el = [[0.0, 0.0, 0.0]], []
    for r in range(rings):
        z = 0.3 if r == 0 else -0.3
        pole = len(pts)
        pts.append([0.0, 0.0, 2 * z])
        th = 2 * np.pi * (np.arange(k) + 0.5 * r) / k
        ring = len(pts)
        pts += [[np.cos(t), np.sin(t), z] for t in th]
        el += [[0, pole, ring + i, ring + (i + 1) % k] for i in range(k)]
    return np.ascontiguousarray(np.array(pts)), np.array(el, np.int32)


@pytest.mark.parametrize("element", [RT0, NED0], ids=["rt0", "ne0"])
@pytest.mark.parametrize("k,rings", [(9, 1), (20, 1), (15, 2)], ids=["k9", "k20", "k15x2"])
def test_edge_ring_parity(element, k, rings):
    """NE0 3D fan enumeration (dofs.cu k_fill_fan3): k = 20 keeps node 0's
    fan within the 24 fixed slots but its 21 larger neighbours beyond the
    register lists (the fan-mode generic path, records built from the fan);
    two rings of 15 overflow the slots (the on-device record fallback);
    k = 9 the register path with a row of 9 tets (row_generic in the
    numeric kernel)."""
    pts, el = edge_ring_mesh(k, rings)
    _check(3, element, pts, el, f"edge ring k={k} x{rings}")


def test_edge_ring_capacity_reported():
    """An NE0-3D row whose tets have more than 21 link vertices exceeds
    row_generic's per-thread list (|W| <= 23): EFEM_ECAPACITY, not wrong values
    and not a non-conformity report."""
    from paper_1409_4618_b200 import _lib, api
    pts, el = edge_ring_mesh(30)
    asm = api.Assembler(torch.from_numpy(pts).cuda(), torch.from_numpy(el).cuda(), NED0)
    with pytest.raises(_lib.EfemError) as ex:
        asm.assemble()
    assert ex.value.status == -8  # EFEM_ECAPACITY (include/efem.h)
