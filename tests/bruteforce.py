"""Brute-force physical-space assembly used to PIN the oracle (pin P7).

Independent of the oracle and of the paper's reference-element machinery: no
reference basis, no Piola map, no quadrature table.  For each physical element
the local basis is built by DOF duality directly in physical coordinates:

  * polynomial space R (affine-invariant, PAPER.md:196-204 / 250-257):
      RT : span{e_1..e_d, x}                     (d+1 functions)
      NE2: span{e_1, e_2, (-x_2, x_1)}           (3)
      NE3: span{e_1, e_2, e_3, e_i x x}          (6)
  * DOF functionals on the GLOBAL entity with the GLOBAL orientation
    (orientation readings C5/C6 in DESIGN.md):
      NE : integral of u . t over the edge, t the unit tangent from the lower
           to the higher global node  -> u(mid) . (x_hi - x_lo)  (exact, u linear)
      RT2: integral of u . nu, nu = clockwise rotation of the unit tangent
           -> u(mid) . rot_cw(x_hi - x_lo)
      RT3: integral of u . nu over the face, nu along (x_b-x_a) x (x_c-x_a),
           a<b<c global -> u(centroid) . ((x_b-x_a) x (x_c-x_a)) / 2
  * integrals of products of affine fields by the simplex moment identities
      int_K 1 = |K|,  int_K x = |K| c,  int_K x x^T = |K|/((d+1)(d+2)) (sum x_i x_i^T + s s^T)
    (s = sum of vertices), exact for the degree-2 integrands here.
  * global numbering: rank of the sorted node tuple in lexicographic order.

Works in float64 (numpy) or exactly in fractions.Fraction (``exact=True``).
"""
from __future__ import annotations

from fractions import Fraction
from itertools import combinations

import numpy as np

RT0, NED0 = 0, 1


def _zeros(shape, exact):
    if exact:
        if isinstance(shape, int):
            return [Fraction(0)] * shape
        return [[Fraction(0)] * shape[1] for _ in range(shape[0])]
    return np.zeros(shape)


def _solve(A, B, exact):
    """Solve A X = B (A m x m)."""
    if not exact:
        return np.linalg.solve(np.array(A, float), np.array(B, float))
    m = len(A)
    M = [list(A[i]) + list(B[i]) for i in range(m)]
    for c in range(m):
        p = next(r for r in range(c, m) if M[r][c] != 0)
        M[c], M[p] = M[p], M[c]
        piv = M[c][c]
        M[c] = [v / piv for v in M[c]]
        for r in range(m):
            if r != c and M[r][c] != 0:
                f = M[r][c]
                M[r] = [a - f * b for a, b in zip(M[r], M[c])]
    return [row[m:] for row in M]


def _poly_space(dim, element):
    """Return list of (a, A) with p(x) = a + A x, as nested lists of ints."""
    d = dim
    I = [[1 if r == c else 0 for c in range(d)] for r in range(d)]
    Z = [[0] * d for _ in range(d)]
    out = [(I[i], Z) for i in range(d)]
    if element == RT0:
        out.append(([0] * d, I))
    elif d == 2:
        out.append(([0, 0], [[0, -1], [1, 0]]))  # (-x2, x1)
    else:
        # e_i x x as a matrix acting on x
        out.append(([0, 0, 0], [[0, 0, 0], [0, 0, -1], [0, 1, 0]]))  # e1 x x = (0,-x3,x2)
        out.append(([0, 0, 0], [[0, 0, 1], [0, 0, 0], [-1, 0, 0]]))  # e2 x x = (x3,0,-x1)
        out.append(([0, 0, 0], [[0, -1, 0], [1, 0, 0], [0, 0, 0]]))  # e3 x x = (-x2,x1,0)
    return out


def _entities(dim, element, g):
    """Global entities of one element as sorted local-vertex tuples ordered by
    global id (local positions)."""
    nv = dim + 1
    size = 3 if (dim == 3 and element == RT0) else 2
    ents = []
    for loc in combinations(range(nv), size):
        ents.append(tuple(sorted(loc, key=lambda i: g[i])))
    return ents


def _cross(u, v):
    return [u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]]


def _det(B):
    if len(B) == 2:
        return B[0][0] * B[1][1] - B[0][1] * B[1][0]
    return (B[0][0] * (B[1][1] * B[2][2] - B[1][2] * B[2][1]) - B[0][1] * (B[1][0] * B[2][2] - B[1][2] * B[2][0])
            + B[0][2] * (B[1][0] * B[2][1] - B[1][1] * B[2][0]))


def element_matrices(dim, element, X, g, exact=False):
    """X: (d+1) x d vertex coords (list or array), g: global ids.
    Returns (keys, M, K) with keys the global node tuples of the local basis."""
    d = dim
    nv = d + 1
    conv = Fraction if exact else float
    X = [[conv(X[i][c]) for c in range(d)] for i in range(nv)]
    B = [[X[c + 1][r] - X[0][r] for c in range(d)] for r in range(d)]
    vol = abs(_det(B)) / (2 if d == 2 else 6)
    polys = _poly_space(d, element)
    m = len(polys)
    ents = _entities(d, element, g)
    assert len(ents) == m

    def evalp(p, x):
        a, A = p
        return [a[r] + sum(A[r][c] * x[c] for c in range(d)) for r in range(d)]

    V = _zeros((m, m), exact)
    for i, loc in enumerate(ents):
        pts = [X[j] for j in loc]
        if len(loc) == 2:
            mid = [(pts[0][c] + pts[1][c]) / 2 for c in range(d)]
            tvec = [pts[1][c] - pts[0][c] for c in range(d)]  # low -> high global
            if element == NED0:
                w = tvec
            else:
                w = [tvec[1], -tvec[0]]  # clockwise rotation (2D RT)
            x_eval = mid
        else:
            x_eval = [(pts[0][c] + pts[1][c] + pts[2][c]) / 3 for c in range(3)]
            u = [pts[1][c] - pts[0][c] for c in range(3)]
            v = [pts[2][c] - pts[0][c] for c in range(3)]
            w = [z / 2 for z in _cross(u, v)]
        for j, p in enumerate(polys):
            pv = evalp(p, x_eval)
            V[i][j] = sum(pv[c] * w[c] for c in range(d))
    Iden = [[conv(1) if r == c else conv(0) for c in range(m)] for r in range(m)]
    C = _solve(V, Iden, exact)  # column k = coefficients of phi_k

    # phi_k = a_k + A_k x
    phis = []
    for k in range(m):
        a = [sum(C[j][k] * polys[j][0][r] for j in range(m)) for r in range(d)]
        A = [[sum(C[j][k] * polys[j][1][r][c] for j in range(m)) for c in range(d)] for r in range(d)]
        phis.append((a, A))
    ssum = [sum(X[i][c] for i in range(nv)) for c in range(d)]
    cen = [s / nv for s in ssum]
    XX = [[(sum(X[i][r] * X[i][c] for i in range(nv)) + ssum[r] * ssum[c]) * vol / ((d + 1) * (d + 2))
           for c in range(d)] for r in range(d)]
    M = _zeros((m, m), exact)
    K = _zeros((m, m), exact)
    for k in range(m):
        ak, Ak = phis[k]
        for l in range(m):
            al, Al = phis[l]
            t0 = vol * sum(ak[r] * al[r] for r in range(d))
            t1 = sum((sum(ak[r] * Al[r][c] for r in range(d)) + sum(al[r] * Ak[r][c] for r in range(d))) * cen[c]
                     for c in range(d)) * vol
            t2 = sum(Ak[r][a] * Al[r][b] * XX[a][b] for r in range(d) for a in range(d) for b in range(d))
            M[k][l] = t0 + t1 + t2
            if element == RT0:
                dk = sum(Ak[r][r] for r in range(d))
                dl = sum(Al[r][r] for r in range(d))
                K[k][l] = vol * dk * dl
            elif d == 2:
                ck = Ak[1][0] - Ak[0][1]
                cl = Al[1][0] - Al[0][1]
                K[k][l] = vol * ck * cl
            else:
                ck = [Ak[2][1] - Ak[1][2], Ak[0][2] - Ak[2][0], Ak[1][0] - Ak[0][1]]
                cl = [Al[2][1] - Al[1][2], Al[0][2] - Al[2][0], Al[1][0] - Al[0][1]]
                K[k][l] = vol * sum(ck[r] * cl[r] for r in range(3))
    keys = [tuple(sorted(g[j] for j in loc)) for loc in ents]
    return keys, M, K


def assemble_dense(dim, element, coords, elems, exact=False):
    """Global dense M, K and the sorted entity list (row i <-> ents[i])."""
    ents = set()
    per = []
    for e in range(len(elems)):
        g = [int(v) for v in elems[e]]
        X = [[coords[v][c] for c in range(dim)] for v in g]
        keys, M, K = element_matrices(dim, element, X, g, exact)
        ents.update(keys)
        per.append((keys, M, K))
    ents = sorted(ents)
    idx = {t: i for i, t in enumerate(ents)}
    R = len(ents)
    if exact:
        GM = [[Fraction(0)] * R for _ in range(R)]
        GK = [[Fraction(0)] * R for _ in range(R)]
    else:
        GM = np.zeros((R, R))
        GK = np.zeros((R, R))
    for keys, M, K in per:
        for k, tk in enumerate(keys):
            for l, tl in enumerate(keys):
                GM[idx[tk]][idx[tl]] += M[k][l]
                GK[idx[tk]][idx[tl]] += K[k][l]
    return ents, GM, GK
