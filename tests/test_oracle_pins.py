"""Pins of the CPU oracle against things other than itself (CPU only).

Each test states what fixes the expected value: a passage of PAPER.md, a
closed form, an invariant, or the independent brute-force assembly in
tests/bruteforce.py (physical-space DOF duality, no Piola, no reference basis).
"""
import json
import os
from fractions import Fraction
from itertools import permutations

import numpy as np
import pytest

import bruteforce
from oracle import oracle as ora
from workloads import NED0, RT0, counts

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
KINDS = [(2, RT0), (2, NED0), (3, RT0), (3, NED0)]
KIND_IDS = ["rt0_2d", "ne0_2d", "rt0_3d", "ne0_3d"]

# Reference vertices of the unit triangle / tetrahedron.
REF2 = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
REF3 = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])

# Fig. 1, read off the arrows, 0-based vertices.
FIG1_EDGES_2D = [(1, 2), (2, 0), (0, 1)]  # NE tangents; RT normals are the outward normals of the same edges
FIG1_EDGES_3D = [(0, 1), (0, 2), (0, 3), (1, 2), (2, 3), (3, 1)]
FIG1_FACES_3D = [((0, 1, 2), 3), ((0, 1, 3), 2), ((0, 2, 3), 1), ((1, 2, 3), 0)]  # face, opposite vertex


def test_local_tables_follow_fig1():
    assert [tuple(r) for r in ora.local_table(2, RT0)] == FIG1_EDGES_2D
    assert [tuple(r) for r in ora.local_table(2, NED0)] == FIG1_EDGES_2D
    assert [tuple(r) for r in ora.local_table(3, NED0)] == FIG1_EDGES_3D
    assert [((r[0], r[1], r[2]), r[3]) for r in ora.local_table(3, RT0)] == FIG1_FACES_3D


def _dof_matrix(dim, element):
    """alpha_hat_i(eta_hat_j), PAPER.md:216-227 (RT) and 271-274 (Ned): integrals
    of the normal / tangential component over edge or face i.  The integrands
    are affine, so the midpoint (centroid) value times the measure is exact."""
    m = ora.n_local_dofs(dim, element)
    A = np.zeros((m, m))
    V = REF2 if dim == 2 else REF3
    for i in range(m):
        if dim == 3 and element == RT0:
            (a, b, c), o = FIG1_FACES_3D[i]
            x = (V[a] + V[b] + V[c]) / 3
            nrm = np.cross(V[b] - V[a], V[c] - V[a])
            area = 0.5 * np.linalg.norm(nrm)
            nrm = nrm / np.linalg.norm(nrm)
            if np.dot(nrm, V[a] - V[o]) < 0:
                nrm = -nrm  # outward (Fig. 1 arrows point outward)
            w = area * nrm
        else:
            s, e = (FIG1_EDGES_2D if dim == 2 else FIG1_EDGES_3D)[i]
            x = (V[s] + V[e]) / 2
            t = V[e] - V[s]  # length * unit tangent
            if element == NED0:
                w = t
            else:  # 2D RT: outward normal of edge i, times its length
                nrm = np.array([t[1], -t[0]])
                opp = 3 - s - e
                if np.dot(nrm, V[s] - V[opp]) < 0:
                    nrm = -nrm
                w = nrm
        val, _ = ora.ref_basis(dim, element, x)
        A[i] = val @ w
    return A


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_kronecker_property(dim, element):
    """alpha_hat_i(eta_hat_j) = delta_ij.  For 3D RT this
    holds for 2x the printed basis (reading C1)."""
    A = _dof_matrix(dim, element)
    np.testing.assert_allclose(A, np.eye(A.shape[0]), atol=1e-15)


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_div_curl_tables_match_finite_differences(dim, element):
    """div / curl tables of ref_basis against central differences of its own
    values (the basis is affine, so differences are exact up to rounding)."""
    rng = np.random.default_rng(7)
    x = rng.random(dim) * 0.3
    h = 0.25
    val0, dc = ora.ref_basis(dim, element, x)
    J = np.zeros((val0.shape[0], dim, dim))  # J[k, comp, deriv]
    for c in range(dim):
        xp, xm = x.copy(), x.copy()
        xp[c] += h
        xm[c] -= h
        vp, _ = ora.ref_basis(dim, element, xp)
        vm, _ = ora.ref_basis(dim, element, xm)
        J[:, :, c] = (vp - vm) / (2 * h)
    if element == RT0:
        np.testing.assert_allclose(dc[:, 0], np.trace(J, axis1=1, axis2=2), atol=1e-13)
    elif dim == 2:
        np.testing.assert_allclose(dc[:, 0], J[:, 1, 0] - J[:, 0, 1], atol=1e-13)
    else:
        curl = np.stack([J[:, 2, 1] - J[:, 1, 2], J[:, 0, 2] - J[:, 2, 0], J[:, 1, 0] - J[:, 0, 1]], axis=1)
        np.testing.assert_allclose(dc, curl, atol=1e-13)


@pytest.mark.parametrize("dim", [2, 3])
def test_quadrature_exact_to_degree_2(dim):
    """int_{K_hat} x^a = a! d! / (|a|+d)! * |K_hat| ... closed form for monomials
    on the unit simplex: prod(a_i!) / (|a| + d)!."""
    from math import factorial

    pts, w = ora.quadrature(dim)
    exps = [e for e in np.ndindex(*(3,) * dim) if sum(e) <= 2]
    for e in exps:
        exact = np.prod([factorial(a) for a in e]) / factorial(sum(e) + dim)
        approx = float(np.sum(w * np.prod(pts ** np.array(e), axis=1)))
        assert abs(approx - exact) < 1e-15, (e, approx, exact)


def _dense_oracle(dim, element, coords, elems):
    A = ora.assemble(dim, element, coords, elems)
    M, K = A.dense()
    return A, M, K


def _n1_mesh(dim):
    coords, elems = ora.build_mesh(dim, 1, 0.0, 0)
    return coords, elems


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_oracle_equals_exact_bruteforce_on_unit_mesh(dim, element):
    """Pin P3/P7: unjittered n=1 mesh (2 triangles / 6 Kuhn tets), exact
    rational brute force vs oracle."""
    coords, elems = _n1_mesh(dim)
    A, M, K = _dense_oracle(dim, element, coords, elems)
    ents, GM, GK = bruteforce.assemble_dense(dim, element, coords.tolist(), elems.tolist(), exact=True)
    assert [tuple(int(v) for v in r) for r in A.dofs2nodes] == [tuple(t) for t in ents]
    GMf = np.array([[float(v) for v in row] for row in GM])
    GKf = np.array([[float(v) for v in row] for row in GK])
    np.testing.assert_allclose(M, GMf, atol=2e-15)
    np.testing.assert_allclose(K, GKf, atol=1e-14)


def test_p3_unit_square_exact_values():
    """SURVEY.md §8(c) P3 (derived from PAPER.md:335-342 by hand): the 2D n=1
    matrices, identical for RT0 and NE0.  Checked against the exact brute force
    AND the oracle (two routes)."""
    F = Fraction
    M = [[F(1, 3), 0, 0, F(-1, 6), 0], [0, F(1, 3), 0, 0, F(-1, 6)], [0, 0, F(1, 3), 0, 0],
         [F(-1, 6), 0, 0, F(1, 3), 0], [0, F(-1, 6), 0, 0, F(1, 3)]]
    K = [[2, 0, -2, 2, 0], [0, 2, -2, 0, 2], [-2, -2, 4, -2, -2], [2, 0, -2, 2, 0], [0, 2, -2, 0, 2]]
    coords, elems = _n1_mesh(2)
    for element in (RT0, NED0):
        ents, GM, GK = bruteforce.assemble_dense(2, element, coords.tolist(), elems.tolist(), exact=True)
        assert ents == [(0, 1), (0, 2), (0, 3), (1, 3), (2, 3)]
        assert GM == [[F(v) for v in r] for r in M]
        assert GK == [[F(v) for v in r] for r in K]
        _, Mo, Ko = _dense_oracle(2, element, coords, elems)
        np.testing.assert_allclose(Mo, np.array(M, dtype=float), atol=1e-15)
        np.testing.assert_allclose(Ko, np.array(K, dtype=float), atol=1e-14)
        # structural zeros are kept (reading C9): 2 x 9 local entries, the
        # shared diagonal counted once -> 17, of which 8 are zeros of M (up to
        # quadrature rounding)
        A = ora.assemble(2, element, coords, elems)
        assert A.col_idx.shape[0] == 17
        assert int(np.sum(np.abs(A.vals_M) < 1e-15)) == 8


def _random_small_mesh(dim, rng, n_elems):
    """n=1 structured mesh, every node jittered (boundary too), node ids
    randomly relabelled, every element's vertex order randomly permuted, then
    the first n_elems elements kept."""
    coords, elems = _n1_mesh(dim)
    coords = coords + rng.uniform(-0.12, 0.12, coords.shape)
    perm = rng.permutation(coords.shape[0])
    inv = np.argsort(perm)
    coords = coords[perm]
    elems = inv[elems].astype(np.int32)
    for e in range(elems.shape[0]):
        elems[e] = elems[e][rng.permutation(dim + 1)]
    return coords, elems[:n_elems]


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
@pytest.mark.parametrize("n_elems", [1, 2, 3, 4])
def test_oracle_equals_bruteforce_random(dim, element, n_elems):
    """Pin P7: 1-4 random elements, random vertex order and node labels."""
    rng = np.random.default_rng(100 * dim + 10 * element + n_elems)
    for trial in range(3):
        coords, elems = _random_small_mesh(dim, rng, n_elems)
        # keep only nodes that are used, renumbered (the oracle only sees the
        # elements; unused nodes are allowed)
        A, M, K = _dense_oracle(dim, element, coords, elems)
        ents, GM, GK = bruteforce.assemble_dense(dim, element, coords, elems)
        assert [tuple(int(v) for v in r) for r in A.dofs2nodes] == [tuple(t) for t in ents]
        np.testing.assert_allclose(M, GM, rtol=0, atol=1e-12 * np.abs(GM).max())
        np.testing.assert_allclose(K, GK, rtol=0, atol=1e-12 * np.abs(GK).max())


def _gradient_incidence(edges, n_nodes):
    G = np.zeros((len(edges), n_nodes))
    for i, (a, b) in enumerate(edges):
        G[i, a] = -1.0
        G[i, b] = 1.0
    return G


@pytest.mark.parametrize("dim,n", [(2, 4), (3, 2)])
def test_de_rham_kernel_ne(dim, n):
    """north_star: curl-curl . G = 0 for the node-to-edge gradient incidence."""
    coords, elems = ora.build_mesh(dim, n, 0.2 if dim == 2 else 0.15, 11)
    A, M, K = _dense_oracle(dim, NED0, coords, elems)
    G = _gradient_incidence(A.dofs2nodes, coords.shape[0])
    assert np.abs(K @ G).max() < 1e-11 * np.abs(K).max()
    # dim ker K^NE = #N - 1 on a contractible domain
    ev = np.linalg.eigvalsh(K)
    assert int(np.sum(ev < 1e-9 * ev.max())) == coords.shape[0] - 1


def test_de_rham_kernel_rt3():
    """K^RT3 C = 0 for the edge-to-face incidence (boundary a->b->c->a)."""
    coords, elems = ora.build_mesh(3, 2, 0.15, 12)
    A, M, K = _dense_oracle(3, RT0, coords, elems)
    E = ora.assemble(3, NED0, coords, elems).dofs2nodes
    eid = {tuple(r): i for i, r in enumerate(E.tolist())}
    C = np.zeros((A.n_dofs, len(E)))
    for f, (a, b, c) in enumerate(A.dofs2nodes.tolist()):
        C[f, eid[(a, b)]] += 1.0
        C[f, eid[(b, c)]] += 1.0
        C[f, eid[(a, c)]] -= 1.0
    assert np.abs(K @ C).max() < 1e-10 * np.abs(K).max()
    ev = np.linalg.eigvalsh(K)
    assert int(np.sum(ev < 1e-9 * ev.max())) == A.n_dofs - elems.shape[0]  # dim ker = #F - #T


def _constant_field_dofs(dim, element, coords, dofs2nodes, v):
    c = np.zeros(dofs2nodes.shape[0])
    for i, t in enumerate(dofs2nodes):
        if element == NED0:
            c[i] = np.dot(coords[t[1]] - coords[t[0]], v)
        elif dim == 2:
            d = coords[t[1]] - coords[t[0]]
            c[i] = np.dot(np.array([d[1], -d[0]]), v)
        else:
            nu = np.cross(coords[t[1]] - coords[t[0]], coords[t[2]] - coords[t[0]])
            c[i] = 0.5 * np.dot(nu, v)
    return c


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_constant_field_interpolant(dim, element):
    """north_star: c^T M c = |v|^2 |Omega| (|Omega| = 1) and K c = 0 for the
    interpolant c of a constant field v; pins normalisation (reading C1),
    signs and the Piola maps on a jittered mesh with mixed det signs (3D)."""
    n = 4 if dim == 2 else 2
    coords, elems = ora.build_mesh(dim, n, 0.2 if dim == 2 else 0.15, 5)
    A, M, K = _dense_oracle(dim, element, coords, elems)
    rng = np.random.default_rng(3)
    v = rng.normal(size=dim)
    c = _constant_field_dofs(dim, element, coords, A.dofs2nodes, v)
    assert abs(c @ M @ c - v @ v) < 1e-13 * (v @ v)
    assert np.abs(K @ c).max() < 1e-11 * np.abs(K).max()


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_spd_psd_symmetry(dim, element):
    n = 4 if dim == 2 else 2
    coords, elems = ora.build_mesh(dim, n, 0.2 if dim == 2 else 0.15, 9)
    A, M, K = _dense_oracle(dim, element, coords, elems)
    assert np.abs(M - M.T).max() <= 1e-15 * np.abs(M).max()
    assert np.abs(K - K.T).max() <= 1e-15 * np.abs(K).max()
    np.linalg.cholesky(M)
    assert np.linalg.eigvalsh(K).min() > -1e-10 * np.abs(K).max()
    if dim == 2 and element == RT0:
        assert int(np.sum(np.linalg.eigvalsh(K) < 1e-9 * np.abs(K).max())) == A.n_dofs - elems.shape[0]


def test_2d_rt_equals_ne():
    """on the same 2D mesh the RT0 and NE0 matrices
    coincide (cof(B) = J^-1 B J with J the 90-degree rotation)."""
    coords, elems = ora.build_mesh(2, 6, 0.2, 21)
    a = ora.assemble(2, RT0, coords, elems)
    b = ora.assemble(2, NED0, coords, elems)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    np.testing.assert_allclose(a.vals_M, b.vals_M, atol=1e-14)
    np.testing.assert_allclose(a.vals_K, b.vals_K, atol=1e-10)


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_vertex_order_invariance(dim, element):
    """Global matrices do not depend on the local vertex order (signs absorb
    it)."""
    n = 3 if dim == 2 else 2
    coords, elems = ora.build_mesh(dim, n, 0.2 if dim == 2 else 0.15, 4)
    a = ora.assemble(dim, element, coords, elems)
    rng = np.random.default_rng(8)
    e2 = elems.copy()
    for e in range(e2.shape[0]):
        e2[e] = e2[e][rng.permutation(dim + 1)]
    b = ora.assemble(dim, element, coords, e2)
    assert np.array_equal(a.dofs2nodes, b.dofs2nodes)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    np.testing.assert_allclose(a.vals_M, b.vals_M, atol=1e-13 * np.abs(a.vals_M).max())
    np.testing.assert_allclose(a.vals_K, b.vals_K, atol=1e-13 * np.abs(a.vals_K).max())


@pytest.mark.parametrize("dim,element,pm,pk", [(2, RT0, 0, -2), (2, NED0, 0, -2), (3, RT0, -1, -3), (3, NED0, 1, -1)],
                         ids=KIND_IDS)
def test_scaling_laws(dim, element, pm, pk):
    """x -> c x scales M by c^pm and K by c^pk (Piola maps)."""
    coords, elems = ora.build_mesh(dim, 2, 0.15, 2)
    a = ora.assemble(dim, element, coords, elems)
    c = 1.7
    b = ora.assemble(dim, element, coords * c, elems)
    np.testing.assert_allclose(b.vals_M, a.vals_M * c ** pm, atol=1e-13 * np.abs(b.vals_M).max())
    np.testing.assert_allclose(b.vals_K, a.vals_K * c ** pk, atol=1e-13 * np.abs(b.vals_K).max())


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_counts_match_closed_forms(dim, element, n):
    if dim == 3 and n == 5:
        n = 4
    coords, elems = ora.build_mesh(dim, n, 0.1, 1)
    A = ora.assemble(dim, element, coords, elems)
    N, T, R, nnz = counts(dim, element, n)
    assert (coords.shape[0], elems.shape[0], A.n_dofs, A.col_idx.shape[0]) == (N, T, R, nnz)


def test_closed_forms_match_paper_tables():
    """Paper-printed sizes (tests/golden/paper_counts.json)."""
    g = json.load(open(os.path.join(GOLDEN, "paper_counts.json")))
    for T, E in g["table5_unit_square_T_E"]["rows"]:
        n = int(round((T / 2) ** 0.5))
        _, T2, E2, _ = counts(2, NED0, n)
        assert (T2, E2) == (T, E)
    for L, F, E in g["table2_unit_cube_F_E"]["rows"]:
        n = 6 * 2 ** (L - 1)
        assert counts(3, RT0, n)[2] == F and counts(3, NED0, n)[2] == E
    for T in g["table3_unit_square_T"]["rows"]:
        n = int(round((T / 2) ** 0.5))
        assert counts(2, RT0, n)[1] == T
    for T in g["table4_unit_cube_T"]["rows"]:
        n = int(round((T / 6) ** (1 / 3)))
        assert counts(3, RT0, n)[1] == T


@pytest.mark.parametrize("L", [1, 2])
def test_oracle_counts_table2(L):
    """Oracle's own enumeration reproduces Table 2."""
    g = json.load(open(os.path.join(GOLDEN, "paper_counts.json")))
    _, F, E = g["table2_unit_cube_F_E"]["rows"][L - 1]
    n = 6 * 2 ** (L - 1)
    coords, elems = ora.build_mesh(3, n, 0.0, 0)
    assert ora.assemble(3, RT0, coords, elems).n_dofs == F
    assert ora.assemble(3, NED0, coords, elems).n_dofs == E


def test_oracle_counts_table5_first_row():
    """Oracle's own enumeration reproduces Table 5 row 1."""
    coords, elems = ora.build_mesh(2, 128, 0.0, 0)
    assert elems.shape[0] == 32768
    assert ora.assemble(2, NED0, coords, elems).n_dofs == 49408


def _dets(dim, coords, elems):
    X = coords[elems]
    B = np.stack([X[:, i + 1] - X[:, 0] for i in range(dim)], axis=2)
    return np.linalg.det(B)


@pytest.mark.parametrize("dim,n,alpha", [(2, 16, 0.1), (2, 9, 0.2), (3, 5, 0.15), (3, 4, 0.2)])
def test_mesh_generator(dim, n, alpha):
    """Input recipe: boundary nodes on the grid, |Omega| = 1,
    every det keeps the sign of the unjittered element, |jitter| <= alpha h,
    deterministic in the seed."""
    c0, e0 = ora.build_mesh(dim, n, 0.0, 3)
    c1, e1 = ora.build_mesh(dim, n, alpha, 3)
    assert np.array_equal(e0, e1)
    grid = np.stack(np.meshgrid(*[np.arange(n + 1) / n] * dim, indexing="ij"), -1)
    grid = grid.transpose(*range(dim)[::-1], dim).reshape(-1, dim)  # node id = i + (n+1) j (+ ...)
    assert np.array_equal(c0, grid)
    bnd = np.any((grid == 0) | (grid == 1), axis=1)
    assert np.array_equal(c1[bnd], grid[bnd])
    assert np.abs(c1 - grid).max() <= alpha / n
    assert np.all(np.abs(c1[~bnd] - grid[~bnd]) > 0)
    d0, d1 = _dets(dim, c0, e0), _dets(dim, c1, e1)
    assert np.all(np.sign(d0) == np.sign(d1))
    fact = 2 if dim == 2 else 6
    assert abs(np.abs(d1).sum() / fact - 1.0) < 1e-12
    c2, _ = ora.build_mesh(dim, n, alpha, 3)
    c3, _ = ora.build_mesh(dim, n, alpha, 4)
    assert np.array_equal(c1, c2) and not np.array_equal(c1, c3)
    if dim == 3:
        assert (d0 > 0).any() and (d0 < 0).any()  # mixed orientations exercise the signs


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
def test_sampled_rows_match_full(dim, element):
    """ora_rows_by_entity (used at full BASELINE sizes) agrees with the full
    assembly row by row."""
    n = 5 if dim == 2 else 3
    coords, elems = ora.build_mesh(dim, n, 0.15, 6)
    A = ora.assemble(dim, element, coords, elems)
    rows = np.array([0, 1, A.n_dofs // 2, A.n_dofs - 1])
    res = ora.rows_by_entity(dim, element, coords, elems, A.dofs2nodes[rows])
    for r, (cols, vm, vk) in zip(rows, res):
        lo, hi = A.row_ptr[r], A.row_ptr[r + 1]
        want_cols = A.dofs2nodes[A.col_idx[lo:hi]]
        assert np.array_equal(cols[:, : want_cols.shape[1]], want_cols)
        assert np.array_equal(vm, A.vals_M[lo:hi]) and np.array_equal(vk, A.vals_K[lo:hi])


def test_oracle_rejects_degenerate_and_bad_input():
    coords = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]])
    with pytest.raises(ValueError):
        ora.assemble(2, RT0, coords, np.array([[0, 1, 2]], np.int32))
    with pytest.raises(ValueError):
        ora.assemble(2, RT0, coords, np.array([[0, 1, 3]], np.int32))


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
@pytest.mark.parametrize("threads,blocks", [(1, 1), (2, 5), (4, 37)])
def test_blocked_equals_serial(dim, element, threads, blocks):
    """The row-range form (ora_assemble_blocked: node ranges -> contiguous
    DOF blocks, each summing its rows in ascending element order) is bitwise
    the serial oracle, on a permuted unstructured-order mesh too (random node
    labels and element order, so block boundaries cut rows anywhere)."""
    n = 9 if dim == 2 else 3
    c, e = ora.build_mesh(dim, n, 0.2 if dim == 2 else 0.15, 21)
    rng = np.random.default_rng(dim * 7 + element)
    perm = rng.permutation(c.shape[0])
    c = np.ascontiguousarray(c[perm])
    e = np.ascontiguousarray(np.argsort(perm)[e][rng.permutation(e.shape[0])].astype(np.int32))
    a = ora.assemble(dim, element, c, e)
    b = ora.assemble(dim, element, c, e, threads=threads, blocks=blocks)
    for f in ("dofs2nodes", "elems2dofs", "signs", "row_ptr", "col_idx", "vals_M", "vals_K"):
        assert getattr(a, f).tobytes() == getattr(b, f).tobytes(), f


def test_blocked_rejects_degenerate():
    c, e = ora.build_mesh(2, 4, 0.0, 0)
    c = c.copy()
    c[e[13][2]] = 0.5 * (c[e[13][0]] + c[e[13][1]])
    with pytest.raises(ValueError):
        ora.assemble(2, NED0, c, e, threads=3)
