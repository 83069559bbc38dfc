/*
 * efem_oracle.cpp -- CPU ORACLE for RT0 / NE0 mass + stiffness assembly.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_1409_4618_b200/) may include, link or call this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load liboracle.so.  It shares no code, header, table or
 * constant with the CUDA path.
 *
 * Plain, slow, obviously-correct: a serial per-element loop that follows the
 * paper (Anjam & Valdman, arXiv:1409.4618; "PAPER.md:N" = line N of the LaTeX
 * source) in its own order and notation:
 *
 *   - reference bases as printed            PAPER.md:228-238 (RT), 275-289 (Ned)
 *     (3D RT: 2x the printed formula, reading C1 in DESIGN.md)
 *   - Piola maps
 *   - sign data
 *   - local matrices                        PAPER.md:344-363 (Eq. RT0local2 ...)
 *     evaluated with the quadrature loop of PAPER.md:671-696 over ALL (k,l)
 *     (no upper-triangle mirror, so the oracle stays independent)
 *   - global matrices M_ij, K_ij
 *   - DOF numbering = rows of edges2nodes / faces2nodes, PAPER.md:369-386;
 *     the row order is lexicographic in sorted node tuples (reading C10)
 *   - accumulation in a std::map in element order, then k, then l, CSR emit.
 *
 * Floating point: fp64, compiled with -ffp-contract=off (no FMA contraction).
 * Parity pins for every function: tests/test_oracle_pins.py.
 */
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <thread>
#include <utility>
#include <vector>

namespace {

enum { ORA_RT0 = 0, ORA_NED0 = 1 };
enum { ORA_OK = 0, ORA_EINVAL = -1, ORA_EDEGENERATE = -2 };

/* ---------------------------------------------------------------------------
 * Seeded structured mesh (input generator; reading C10 in DESIGN.md).
 * Node id = i + (n+1) j (+ (n+1)^2 k).  Interior nodes are jittered per axis
 * by (2u-1)*(alpha/n), u = (H(seed, node*d+axis) >> 11) * 2^-53 with H a
 * SplitMix64 counter hash.  Boundary nodes stay on the grid, so |Omega| = 1.
 * ------------------------------------------------------------------------- */
uint64_t counter_hash(uint64_t seed, uint64_t idx) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (idx + 1ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

double grid_coord(int i, int n, bool interior, double alpha, uint64_t seed, uint64_t hidx) {
    double x = (double)i / (double)n;
    if (!interior) return x;
    double u = (double)(counter_hash(seed, hidx) >> 11) * 0x1.0p-53;
    double t = 2.0 * u;
    t = t - 1.0;
    double h = alpha / (double)n;
    double off = t * h;
    return x + off;
}

/* ---------------------------------------------------------------------------
 * Reference element tables (Fig. 1, lines 54-157), 0-based.
 * Edge k runs start -> end (the tangent direction drawn in Fig. 1).
 * Face k is given by its three vertices and the opposite vertex.
 * ------------------------------------------------------------------------- */
const int EDGES2D[3][2] = {{1, 2}, {2, 0}, {0, 1}};
const int EDGES3D[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {2, 3}, {3, 1}};
const int FACES3D[4][4] = {{0, 1, 2, 3}, {0, 1, 3, 2}, {0, 2, 3, 1}, {1, 2, 3, 0}};

int n_local_dofs(int dim, int element) {
    if (dim == 2) return 3;
    return element == ORA_RT0 ? 4 : 6;
}

/* Reference basis functions at xh, exactly as printed.
 *   val[k*dim + c]  = c-th component of eta_hat_{k+1}(xh)
 *   dc[k*nc + c]    = div eta_hat (nc=1), 2D curl (nc=1) or 3D curl (nc=3)
 * RT 2D:  PAPER.md:230-232.  RT 3D: PAPER.md:235-238 times 2 (reading C1).
 * Ned 2D: PAPER.md:277-279.  Ned 3D: PAPER.md:282-289.
 * The div / curl entries are the derivatives of the printed polynomials,
 * computed by hand from them (div(x1,x2)=2, curl(-x2,x1)=2, ...). */
void ref_basis(int dim, int element, const double* xh, double* val, double* dc) {
    const double x1 = xh[0], x2 = xh[1], x3 = dim == 3 ? xh[2] : 0.0;
    if (dim == 2 && element == ORA_RT0) {
        const double v[3][2] = {{x1, x2}, {x1 - 1.0, x2}, {x1, x2 - 1.0}};
        for (int k = 0; k < 3; ++k) {
            val[2 * k] = v[k][0];
            val[2 * k + 1] = v[k][1];
            dc[k] = 2.0;
        }
    } else if (dim == 2 && element == ORA_NED0) {
        const double v[3][2] = {{-x2, x1}, {-x2, x1 - 1.0}, {1.0 - x2, x1}};
        for (int k = 0; k < 3; ++k) {
            val[2 * k] = v[k][0];
            val[2 * k + 1] = v[k][1];
            dc[k] = 2.0; /* d1 v2 - d2 v1 = 1 - (-1) */
        }
    } else if (dim == 3 && element == ORA_RT0) {
        const double v[4][3] = {{x1, x2, x3 - 1.0}, {x1, x2 - 1.0, x3}, {x1 - 1.0, x2, x3}, {x1, x2, x3}};
        for (int k = 0; k < 4; ++k) {
            for (int c = 0; c < 3; ++c) val[3 * k + c] = 2.0 * v[k][c];
            dc[k] = 2.0 * 3.0;
        }
    } else {
        const double v[6][3] = {{1.0 - x3 - x2, x1, x1}, {x2, 1.0 - x3 - x1, x2}, {x3, x3, 1.0 - x2 - x1},
                                {-x2, x1, 0.0},          {0.0, -x3, x2},          {x3, 0.0, -x1}};
        /* curl w = (d2 w3 - d3 w2, d3 w1 - d1 w3, d1 w2 - d2 w1) */
        const double c[6][3] = {{0.0 - 0.0, -1.0 - 1.0, 1.0 - (-1.0)},
                                {1.0 - (-1.0), 0.0 - 0.0, -1.0 - 1.0},
                                {-1.0 - 1.0, 1.0 - (-1.0), 0.0 - 0.0},
                                {0.0 - 0.0, 0.0 - 0.0, 1.0 - (-1.0)},
                                {1.0 - (-1.0), 0.0 - 0.0, 0.0 - 0.0},
                                {0.0 - 0.0, 1.0 - (-1.0), 0.0 - 0.0}};
        for (int k = 0; k < 6; ++k)
            for (int cc = 0; cc < 3; ++cc) {
                val[3 * k + cc] = v[k][cc];
                dc[3 * k + cc] = c[k][cc];
            }
    }
}

/* Degree-2 quadrature on the reference element (PAPER.md:648 cites Dunavant
 * for triangles and Zhang-Cui-Liu for tetrahedra; reading C7). */
int quadrature(int dim, double* pts, double* w) {
    if (dim == 2) {
        const double p[3][2] = {{1.0 / 6.0, 1.0 / 6.0}, {2.0 / 3.0, 1.0 / 6.0}, {1.0 / 6.0, 2.0 / 3.0}};
        for (int q = 0; q < 3; ++q) {
            pts[2 * q] = p[q][0];
            pts[2 * q + 1] = p[q][1];
            w[q] = 1.0 / 6.0;
        }
        return 3;
    }
    const double s5 = std::sqrt(5.0);
    const double a = (5.0 - s5) / 20.0, b = (5.0 + 3.0 * s5) / 20.0;
    const double p[4][3] = {{a, a, a}, {b, a, a}, {a, b, a}, {a, a, b}};
    for (int q = 0; q < 4; ++q) {
        for (int c = 0; c < 3; ++c) pts[3 * q + c] = p[q][c];
        w[q] = 1.0 / 24.0;
    }
    return 4;
}

/* Affine map F_K(xh) = B_K xh + b_K, B_K = [p1-p0 | p2-p0 (| p3-p0)] as
 * columns.  B[r][c] row-major. */
double affine(int dim, const double* verts, double B[3][3]) {
    for (int r = 0; r < dim; ++r)
        for (int c = 0; c < dim; ++c) B[r][c] = verts[(c + 1) * dim + r] - verts[r];
    if (dim == 2) return B[0][0] * B[1][1] - B[0][1] * B[1][0];
    return B[0][0] * (B[1][1] * B[2][2] - B[1][2] * B[2][1]) - B[0][1] * (B[1][0] * B[2][2] - B[1][2] * B[2][0]) +
           B[0][2] * (B[1][0] * B[2][1] - B[1][1] * B[2][0]);
}

/* B^{-T} by the adjugate: inv(B) = adj(B)/det, so B^{-T}[r][c] = cof(B)[r][c]/det. */
void inverse_transpose(int dim, const double B[3][3], double det, double BiT[3][3]) {
    if (dim == 2) {
        BiT[0][0] = B[1][1] / det;
        BiT[0][1] = -B[1][0] / det;
        BiT[1][0] = -B[0][1] / det;
        BiT[1][1] = B[0][0] / det;
        return;
    }
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            const int r1 = (r + 1) % 3, r2 = (r + 2) % 3, c1 = (c + 1) % 3, c2 = (c + 2) % 3;
            BiT[r][c] = (B[r1][c1] * B[r2][c2] - B[r1][c2] * B[r2][c1]) / det;
        }
}

/* Local matrices M^K, K^K (full m x m, row-major), PAPER.md:344-363 with the
 * sign typo at PAPER.md:361 read as s_k s_l (reading C2).  Every integral is
 * the degree-2 quadrature sum over the reference element, as in the listing
 * at PAPER.md:671-696 (there intquad(1) for the constant stiffness integrand;
 * the degree-2 rule gives the same integral). */
int local_matrices(int dim, int element, const double* verts, const int* s, double* M, double* K) {
    double B[3][3];
    const double det = affine(dim, verts, B);
    if (!(det != 0.0) || !std::isfinite(det)) return ORA_EDEGENERATE;
    const double adet = std::fabs(det);
    double BiT[3][3];
    inverse_transpose(dim, B, det, BiT);
    const int m = n_local_dofs(dim, element);
    const int nc = (dim == 3 && element == ORA_NED0) ? 3 : 1;
    double pts[12], w[4];
    const int nip = quadrature(dim, pts, w);
    for (int i = 0; i < m * m; ++i) M[i] = K[i] = 0.0;
    for (int q = 0; q < nip; ++q) {
        double val[18], dc[18], mapped[6][3], dmapped[6][3];
        ref_basis(dim, element, pts + dim * q, val, dc);
        for (int k = 0; k < m; ++k) {
            for (int r = 0; r < dim; ++r) {
                double acc = 0.0;
                for (int c = 0; c < dim; ++c)
                    acc += (element == ORA_RT0 ? B[r][c] : BiT[r][c]) * val[k * dim + c];
                mapped[k][r] = acc; /* RT: B eta_hat; Ned: B^{-T} eta_hat */
            }
            if (nc == 3) {
                for (int r = 0; r < 3; ++r) {
                    double acc = 0.0;
                    for (int c = 0; c < 3; ++c) acc += B[r][c] * dc[3 * k + c];
                    dmapped[k][r] = acc; /* B curl_hat */
                }
            } else {
                dmapped[k][0] = dc[k]; /* div_hat or 2D curl_hat */
            }
        }
        for (int k = 0; k < m; ++k)
            for (int l = 0; l < m; ++l) {
                double vv = 0.0;
                for (int r = 0; r < dim; ++r) vv += (s[k] * mapped[k][r]) * (s[l] * mapped[l][r]);
                double dd = 0.0;
                for (int r = 0; r < nc; ++r) dd += (s[k] * dmapped[k][r]) * (s[l] * dmapped[l][r]);
                M[k * m + l] += w[q] * vv;
                K[k * m + l] += w[q] * dd;
            }
    }
    for (int i = 0; i < m * m; ++i) {
        M[i] = (element == ORA_RT0) ? M[i] / adet : M[i] * adet; /* PAPER.md:345 vs 353 */
        K[i] = K[i] / adet;
    }
    return ORA_OK;
}

/* Global entity (edge / face) of local DOF k as a sorted node tuple;
 * unused trailing slot = -1. */
std::array<int, 3> entity_key(int dim, int element, const int32_t* g, int k) {
    std::array<int, 3> t{-1, -1, -1};
    if (dim == 3 && element == ORA_RT0) {
        int a = g[FACES3D[k][0]], b = g[FACES3D[k][1]], c = g[FACES3D[k][2]];
        int v[3] = {a, b, c};
        std::sort(v, v + 3);
        t = {v[0], v[1], v[2]};
    } else {
        const int(*E)[2] = dim == 2 ? EDGES2D : EDGES3D;
        int a = g[E[k][0]], b = g[E[k][1]];
        t = {std::min(a, b), std::max(a, b), -1};
    }
    return t;
}

/* Sign data (2D rule PAPER.md:528; 3D rules: readings C3,
 * C5, C6).  Edges: +1 iff the local start node has the lower global id, i.e.
 * the global tangent runs from the lower to the higher global node.  Faces:
 * the global normal is nu = (x_b - x_a) x (x_c - x_a) for global ids a<b<c;
 * the Piola-mapped local function carries outward flux sign(det B_K)
 * (PAPER.md:317-321), so s = sign(det B_K) * sign(nu . (x_a - x_opp)). */
int sign_of(int dim, int element, const int32_t* g, const double* verts, int k) {
    if (dim == 3 && element == ORA_RT0) {
        double B[3][3];
        const double det = affine(3, verts, B);
        int loc[3] = {FACES3D[k][0], FACES3D[k][1], FACES3D[k][2]};
        std::sort(loc, loc + 3, [&](int p, int q) { return g[p] < g[q]; });
        const double* xa = verts + 3 * loc[0];
        const double* xb = verts + 3 * loc[1];
        const double* xc = verts + 3 * loc[2];
        const double* xo = verts + 3 * FACES3D[k][3];
        double u[3], v[3], nu[3];
        for (int c = 0; c < 3; ++c) {
            u[c] = xb[c] - xa[c];
            v[c] = xc[c] - xa[c];
        }
        nu[0] = u[1] * v[2] - u[2] * v[1];
        nu[1] = u[2] * v[0] - u[0] * v[2];
        nu[2] = u[0] * v[1] - u[1] * v[0];
        double out = 0.0;
        for (int c = 0; c < 3; ++c) out += nu[c] * (xa[c] - xo[c]);
        const int sdet = det > 0.0 ? 1 : -1;
        const int sout = out > 0.0 ? 1 : -1;
        return sdet * sout;
    }
    const int(*E)[2] = dim == 2 ? EDGES2D : EDGES3D;
    return g[E[k][0]] < g[E[k][1]] ? 1 : -1;
}

struct Result {
    int dim = 0, element = 0, m = 0, ek = 0;
    std::vector<int32_t> dofs2nodes, elems2dofs, row_ptr, col_idx;
    std::vector<int8_t> signs;
    std::vector<double> vals_M, vals_K;
    int64_t bad_element = -1;
};

int validate(int dim, int element, int64_t n_nodes, int64_t n_elems, const int32_t* elems) {
    if (dim != 2 && dim != 3) return ORA_EINVAL;
    if (element != ORA_RT0 && element != ORA_NED0) return ORA_EINVAL;
    if (n_nodes < 0 || n_elems < 0) return ORA_EINVAL;
    for (int64_t e = 0; e < n_elems; ++e)
        for (int v = 0; v <= dim; ++v) {
            int32_t id = elems[e * (dim + 1) + v];
            if (id < 0 || id >= n_nodes) return ORA_EINVAL;
        }
    return ORA_OK;
}

}  // namespace

extern "C" {

int ora_mesh_sizes(int dim, int n, int64_t* n_nodes, int64_t* n_elems) {
    if ((dim != 2 && dim != 3) || n < 1) return ORA_EINVAL;
    const int64_t n1 = n + 1;
    *n_nodes = dim == 2 ? n1 * n1 : n1 * n1 * n1;
    *n_elems = dim == 2 ? 2ll * n * n : 6ll * n * n * n;
    return ORA_OK;
}

int ora_build_mesh(int dim, int n, double alpha, uint64_t seed, double* coords, int32_t* elems) {
    int64_t N, T;
    if (ora_mesh_sizes(dim, n, &N, &T) != ORA_OK) return ORA_EINVAL;
    const int n1 = n + 1;
    if (dim == 2) {
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i <= n; ++i) {
                const int64_t node = i + (int64_t)n1 * j;
                const bool in = i > 0 && i < n && j > 0 && j < n;
                coords[2 * node + 0] = grid_coord(i, n, in, alpha, seed, (uint64_t)node * 2 + 0);
                coords[2 * node + 1] = grid_coord(j, n, in, alpha, seed, (uint64_t)node * 2 + 1);
            }
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                const int64_t c = i + (int64_t)n * j;
                const int32_t v00 = i + n1 * j, v10 = v00 + 1, v01 = v00 + n1, v11 = v01 + 1;
                int32_t* e0 = elems + 6 * c;
                e0[0] = v00; e0[1] = v10; e0[2] = v11;  /* counter-clockwise */
                e0[3] = v00; e0[4] = v11; e0[5] = v01;  /* counter-clockwise */
            }
        return ORA_OK;
    }
    for (int k = 0; k <= n; ++k)
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i <= n; ++i) {
                const int64_t node = i + (int64_t)n1 * (j + (int64_t)n1 * k);
                const bool in = i > 0 && i < n && j > 0 && j < n && k > 0 && k < n;
                coords[3 * node + 0] = grid_coord(i, n, in, alpha, seed, (uint64_t)node * 3 + 0);
                coords[3 * node + 1] = grid_coord(j, n, in, alpha, seed, (uint64_t)node * 3 + 1);
                coords[3 * node + 2] = grid_coord(k, n, in, alpha, seed, (uint64_t)node * 3 + 2);
            }
    /* Kuhn split: 6 tets along the monotone lattice paths (0,0,0)->(1,1,1),
     * axis permutations in lexicographic order. */
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const int64_t stride[3] = {1, n1, (int64_t)n1 * n1};
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                const int64_t c = i + (int64_t)n * (j + (int64_t)n * k);
                const int64_t v0 = i + stride[1] * j + stride[2] * k;
                for (int p = 0; p < 6; ++p) {
                    int32_t* e = elems + 4 * (6 * c + p);
                    int64_t v = v0;
                    e[0] = (int32_t)v;
                    v += stride[perms[p][0]];
                    e[1] = (int32_t)v;
                    v += stride[perms[p][1]];
                    e[2] = (int32_t)v;
                    v += stride[perms[p][2]];
                    e[3] = (int32_t)v;
                }
            }
    return ORA_OK;
}

/* L-shape (0,1)^2 \ (1/2,1)^2 (Table 1 domain) on the m x m
 * grid, m even, h = m/2 (reading L1): cells (i, j) with i >= h and j >= h are
 * dropped, nodes (i, j) with i > h and j > h too; both numbered row-major over
 * what remains; 2 counter-clockwise triangles per cell as ora_build_mesh;
 * jitter on nodes off the L's boundary (including the re-entrant edges). */
int ora_lshape_sizes(int m, int64_t* n_nodes, int64_t* n_elems) {
    if (m < 2 || (m & 1)) return ORA_EINVAL;
    int64_t nn = 0, ne = 0;
    for (int j = 0; j <= m; ++j)
        for (int i = 0; i <= m; ++i)
            if (!(i > m / 2 && j > m / 2)) ++nn;
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i)
            if (!(i >= m / 2 && j >= m / 2)) ne += 2;
    *n_nodes = nn;
    *n_elems = ne;
    return ORA_OK;
}

int ora_build_lshape(int m, double alpha, uint64_t seed, double* coords, int32_t* elems) {
    if (m < 2 || (m & 1)) return ORA_EINVAL;
    const int h = m / 2;
    std::vector<int32_t> id((size_t)(m + 1) * (m + 1), -1);
    int32_t next = 0;
    for (int j = 0; j <= m; ++j)
        for (int i = 0; i <= m; ++i) {
            if (i > h && j > h) continue;
            const int32_t node = next++;
            id[(size_t)j * (m + 1) + i] = node;
            const bool in = i > 0 && i < m && j > 0 && j < m && !(i >= h && j >= h);
            coords[2 * node + 0] = grid_coord(i, m, in, alpha, seed, (uint64_t)node * 2 + 0);
            coords[2 * node + 1] = grid_coord(j, m, in, alpha, seed, (uint64_t)node * 2 + 1);
        }
    int64_t c = 0;
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) {
            if (i >= h && j >= h) continue;
            const int32_t v00 = id[(size_t)j * (m + 1) + i], v10 = id[(size_t)j * (m + 1) + i + 1];
            const int32_t v01 = id[(size_t)(j + 1) * (m + 1) + i], v11 = id[(size_t)(j + 1) * (m + 1) + i + 1];
            int32_t* e = elems + 6 * c;
            e[0] = v00; e[1] = v10; e[2] = v11;
            e[3] = v00; e[4] = v11; e[5] = v01;
            ++c;
        }
    return ORA_OK;
}

int ora_n_local_dofs(int dim, int element) { return n_local_dofs(dim, element); }

int ora_ref_basis(int dim, int element, const double* xh, double* val, double* dc) {
    if ((dim != 2 && dim != 3) || (element != ORA_RT0 && element != ORA_NED0)) return ORA_EINVAL;
    ref_basis(dim, element, xh, val, dc);
    return ORA_OK;
}

int ora_quadrature(int dim, double* pts, double* w) {
    if (dim != 2 && dim != 3) return ORA_EINVAL;
    return quadrature(dim, pts, w);
}

/* Local entity table: for edges out[2k]=start, out[2k+1]=end; for faces
 * out[4k..4k+3] = three face vertices then the opposite vertex. */
int ora_local_table(int dim, int element, int* out) {
    const int m = n_local_dofs(dim, element);
    if (dim == 3 && element == ORA_RT0) {
        for (int k = 0; k < 4; ++k)
            for (int c = 0; c < 4; ++c) out[4 * k + c] = FACES3D[k][c];
    } else {
        const int(*E)[2] = dim == 2 ? EDGES2D : EDGES3D;
        for (int k = 0; k < m; ++k) {
            out[2 * k] = E[k][0];
            out[2 * k + 1] = E[k][1];
        }
    }
    return m;
}

/* One element: verts[(d+1)*d], global ids g[d+1] (for the signs).  Writes the
 * signs s[m] and the full signed local matrices M[m*m], K[m*m]. */
int ora_element(int dim, int element, const double* verts, const int32_t* g, int8_t* s_out, double* M, double* K) {
    if ((dim != 2 && dim != 3) || (element != ORA_RT0 && element != ORA_NED0)) return ORA_EINVAL;
    const int m = n_local_dofs(dim, element);
    int s[6];
    for (int k = 0; k < m; ++k) {
        s[k] = sign_of(dim, element, g, verts, k);
        s_out[k] = (int8_t)s[k];
    }
    return local_matrices(dim, element, verts, s, M, K);
}

/* Whole assembly.  Returns an opaque handle or NULL; *status gets the code. */
void* ora_assemble(int dim, int element, int64_t n_nodes, int64_t n_elems, const double* coords,
                   const int32_t* elems, int* status) {
    *status = validate(dim, element, n_nodes, n_elems, elems);
    if (*status != ORA_OK) return nullptr;
    Result* R = new Result;
    R->dim = dim;
    R->element = element;
    const int m = n_local_dofs(dim, element);
    const int ek = (dim == 3 && element == ORA_RT0) ? 3 : 2;
    R->m = m;
    R->ek = ek;
    const int nv = dim + 1;

    /* DOFs: the set of global entities, numbered by rank. */
    std::set<std::array<int, 3>> ents;
    for (int64_t e = 0; e < n_elems; ++e)
        for (int k = 0; k < m; ++k) ents.insert(entity_key(dim, element, elems + e * nv, k));
    std::map<std::array<int, 3>, int32_t> id;
    int32_t next = 0;
    for (const auto& t : ents) {
        id[t] = next++;
        for (int c = 0; c < ek; ++c) R->dofs2nodes.push_back(t[c]);
    }

    R->elems2dofs.resize((size_t)n_elems * m);
    R->signs.resize((size_t)n_elems * m);
    std::map<std::pair<int32_t, int32_t>, std::pair<double, double>> acc;
    std::vector<double> verts(nv * dim);
    double M[36], K[36];
    int s[6];
    for (int64_t e = 0; e < n_elems; ++e) {
        const int32_t* g = elems + e * nv;
        for (int v = 0; v < nv; ++v)
            for (int c = 0; c < dim; ++c) verts[v * dim + c] = coords[(int64_t)g[v] * dim + c];
        int32_t dof[6];
        for (int k = 0; k < m; ++k) {
            dof[k] = id[entity_key(dim, element, g, k)];
            s[k] = sign_of(dim, element, g, verts.data(), k);
            R->elems2dofs[(size_t)e * m + k] = dof[k];
            R->signs[(size_t)e * m + k] = (int8_t)s[k];
        }
        if (local_matrices(dim, element, verts.data(), s, M, K) != ORA_OK) {
            *status = ORA_EDEGENERATE;
            R->bad_element = e;
            delete R;
            return nullptr;
        }
        for (int k = 0; k < m; ++k)
            for (int l = 0; l < m; ++l) {
                auto& a = acc[{dof[k], dof[l]}];
                a.first += M[k * m + l];
                a.second += K[k * m + l];
            }
    }

    /* CSR emit ("the global matrix is assembled from the local
     * matrices"); every structural entry is kept, zeros included (reading C9). */
    R->row_ptr.assign((size_t)next + 1, 0);
    for (const auto& kv : acc) {
        R->row_ptr[kv.first.first + 1] += 1;
        R->col_idx.push_back(kv.first.second);
        R->vals_M.push_back(kv.second.first);
        R->vals_K.push_back(kv.second.second);
    }
    for (int32_t r = 0; r < next; ++r) R->row_ptr[r + 1] += R->row_ptr[r];
    return R;
}

int ora_result_sizes(void* h, int64_t* n_dofs, int64_t* nnz) {
    Result* R = (Result*)h;
    *n_dofs = (int64_t)R->row_ptr.size() - 1;
    *nnz = (int64_t)R->col_idx.size();
    return ORA_OK;
}

int ora_result_copy(void* h, int32_t* dofs2nodes, int32_t* elems2dofs, int8_t* signs, int32_t* row_ptr,
                    int32_t* col_idx, double* vals_M, double* vals_K) {
    Result* R = (Result*)h;
    auto cp = [](void* dst, const void* src, size_t bytes) {
        if (dst && bytes) std::memcpy(dst, src, bytes);
    };
    cp(dofs2nodes, R->dofs2nodes.data(), R->dofs2nodes.size() * sizeof(int32_t));
    cp(elems2dofs, R->elems2dofs.data(), R->elems2dofs.size() * sizeof(int32_t));
    cp(signs, R->signs.data(), R->signs.size());
    cp(row_ptr, R->row_ptr.data(), R->row_ptr.size() * sizeof(int32_t));
    cp(col_idx, R->col_idx.data(), R->col_idx.size() * sizeof(int32_t));
    cp(vals_M, R->vals_M.data(), R->vals_M.size() * sizeof(double));
    cp(vals_K, R->vals_K.data(), R->vals_K.size() * sizeof(double));
    return ORA_OK;
}

void ora_free(void* h) { delete (Result*)h; }

/* Row-range (block) form of ora_assemble, for full-size parity at every
 * BASELINE config and for the all-core CPU baseline ("a
 * row-range-partitioned OpenMP variant on all nproc host cores; each thread
 * owns a contiguous row range and scans all elements").
 *
 * DOF ids are lexicographic ranks of the sorted node tuples (PAPER.md:386,
 * reading C10), so the entities whose MINIMUM node lies in a node range
 * [lo, hi) are a contiguous block of global DOF ids (= rows).  The node range
 * [0, n_nodes) is cut into n_blocks contiguous ranges; blocks are handed to
 * n_threads threads.  Per block, the same steps as ora_assemble, restricted
 * to the block's rows:
 *   A. scan ALL elements in ascending order; keep those with a local entity
 *      whose minimum node lies in [lo, hi); the block's entity set is the
 *      std::set of those entities
 *   B. (serial) the block's first DOF id = sum of the sizes of the earlier
 *      blocks' sets; dofs2nodes = the sets in block order
 *   C. for the kept elements in ascending order: signs (sign_of), local
 *      matrices (local_matrices, the full m x m quadrature of PAPER.md:344-363),
 *      and for every local DOF k the block owns, row k added into a
 *      std::map<(row, col)> -- column ids looked up in the owning block's set
 *   D. (serial) CSR emit, blocks in order.
 * Every (row, col) entry receives its contributions in ascending element
 * order, as in ora_assemble, so the result is bitwise identical to it
 * (pinned: tests/test_oracle_pins.py::test_blocked_equals_serial). */
void* ora_assemble_blocked(int dim, int element, int64_t n_nodes, int64_t n_elems, const double* coords,
                           const int32_t* elems, int n_threads, int n_blocks, int* status) {
    *status = validate(dim, element, n_nodes, n_elems, elems);
    if (*status != ORA_OK) return nullptr;
    if (n_threads < 1) n_threads = 1;
    if (n_blocks < 1) n_blocks = 1;
    if (n_nodes > 0 && n_blocks > n_nodes) n_blocks = (int)n_nodes;
    const int m = n_local_dofs(dim, element);
    const int ek = (dim == 3 && element == ORA_RT0) ? 3 : 2;
    const int nv = dim + 1;
    std::vector<int64_t> lo(n_blocks + 1);
    for (int b = 0; b <= n_blocks; ++b) lo[b] = n_nodes * b / n_blocks;
    auto block_of = [&](int node) {
        return (int)(std::upper_bound(lo.begin(), lo.end(), (int64_t)node) - lo.begin()) - 1;
    };
    struct Block {
        std::vector<int64_t> elist;
        std::vector<std::array<int, 3>> keys;  // sorted entity set
        int64_t first = 0;
        std::vector<int32_t> row_len, col;
        std::vector<double> vm, vk;
        int64_t bad = -1;
    };
    std::vector<Block> B(n_blocks);
    Result* R = new Result;
    R->dim = dim;
    R->element = element;
    R->m = m;
    R->ek = ek;
    R->elems2dofs.assign((size_t)n_elems * m, -1);
    R->signs.assign((size_t)n_elems * m, 0);

    auto run = [&](auto&& body) {
        std::atomic<int> next{0};
        std::vector<std::thread> pool;
        for (int t = 0; t < n_threads; ++t)
            pool.emplace_back([&] {
                for (int b = next++; b < n_blocks; b = next++) body(b);
            });
        for (auto& th : pool) th.join();
    };

    /* A */
    run([&](int b) {
        Block& blk = B[b];
        std::set<std::array<int, 3>> ents;
        for (int64_t e = 0; e < n_elems; ++e) {
            const int32_t* g = elems + e * nv;
            bool keep = false;
            for (int k = 0; k < m; ++k) {
                const std::array<int, 3> t = entity_key(dim, element, g, k);
                if (t[0] >= lo[b] && t[0] < lo[b + 1]) {
                    ents.insert(t);
                    keep = true;
                }
            }
            if (keep) blk.elist.push_back(e);
        }
        blk.keys.assign(ents.begin(), ents.end());
    });
    /* B */
    int64_t total = 0;
    for (int b = 0; b < n_blocks; ++b) {
        B[b].first = total;
        total += (int64_t)B[b].keys.size();
        for (const auto& t : B[b].keys)
            for (int c = 0; c < ek; ++c) R->dofs2nodes.push_back(t[c]);
    }
    auto dof_of = [&](const std::array<int, 3>& t) -> int64_t {
        const Block& o = B[block_of(t[0])];
        const auto it = std::lower_bound(o.keys.begin(), o.keys.end(), t);
        return o.first + (int64_t)(it - o.keys.begin());
    };
    /* C */
    run([&](int b) {
        Block& blk = B[b];
        std::map<std::pair<int32_t, int32_t>, std::pair<double, double>> acc;
        std::vector<double> verts(nv * dim);
        double M[36], K[36];
        int s[6];
        for (const int64_t e : blk.elist) {
            const int32_t* g = elems + e * nv;
            for (int v = 0; v < nv; ++v)
                for (int c = 0; c < dim; ++c) verts[v * dim + c] = coords[(int64_t)g[v] * dim + c];
            int32_t dof[6];
            bool own[6];
            for (int k = 0; k < m; ++k) {
                const std::array<int, 3> t = entity_key(dim, element, g, k);
                dof[k] = (int32_t)dof_of(t);
                own[k] = t[0] >= lo[b] && t[0] < lo[b + 1];
                s[k] = sign_of(dim, element, g, verts.data(), k);
                if (own[k]) {
                    R->elems2dofs[(size_t)e * m + k] = dof[k];
                    R->signs[(size_t)e * m + k] = (int8_t)s[k];
                }
            }
            if (local_matrices(dim, element, verts.data(), s, M, K) != ORA_OK) {
                blk.bad = e;
                return;
            }
            for (int k = 0; k < m; ++k) {
                if (!own[k]) continue;
                for (int l = 0; l < m; ++l) {
                    auto& a = acc[{dof[k], dof[l]}];
                    a.first += M[k * m + l];
                    a.second += K[k * m + l];
                }
            }
        }
        blk.row_len.assign(blk.keys.size(), 0);
        for (const auto& kv : acc) {
            blk.row_len[kv.first.first - blk.first] += 1;
            blk.col.push_back(kv.first.second);
            blk.vm.push_back(kv.second.first);
            blk.vk.push_back(kv.second.second);
        }
    });
    /* D */
    int64_t bad = -1;
    for (const Block& blk : B)
        if (blk.bad >= 0 && (bad < 0 || blk.bad < bad)) bad = blk.bad;
    if (bad >= 0) {
        *status = ORA_EDEGENERATE;
        delete R;
        return nullptr;
    }
    R->row_ptr.assign((size_t)total + 1, 0);
    size_t nnz = 0;
    for (const Block& blk : B) nnz += blk.col.size();
    R->col_idx.reserve(nnz);
    R->vals_M.reserve(nnz);
    R->vals_K.reserve(nnz);
    for (const Block& blk : B) {
        for (size_t r = 0; r < blk.row_len.size(); ++r)
            R->row_ptr[blk.first + r + 1] = R->row_ptr[blk.first + r] + blk.row_len[r];
        R->col_idx.insert(R->col_idx.end(), blk.col.begin(), blk.col.end());
        R->vals_M.insert(R->vals_M.end(), blk.vm.begin(), blk.vm.end());
        R->vals_K.insert(R->vals_K.end(), blk.vk.begin(), blk.vk.end());
    }
    return R;
}

/* Sampled rows for meshes too large for the full oracle.  For each query
 * entity (sorted node tuple, ek ints, trailing -1 for edges), scan every
 * element once, accumulate the query row keyed by the COLUMN ENTITY tuple
 * (the DOF numbering is not needed), in element order then l.
 * Output per query q: count[q] <= cap entries, sorted by column tuple:
 *   cols[(q*cap + j)*3 + 0..2], vals_M[q*cap + j], vals_K[q*cap + j]. */
int ora_rows_by_entity(int dim, int element, int64_t n_nodes, int64_t n_elems, const double* coords,
                       const int32_t* elems, int64_t n_query, const int32_t* query, int cap, int32_t* count,
                       int32_t* cols, double* vals_M, double* vals_K) {
    int st = validate(dim, element, n_nodes, n_elems, elems);
    if (st != ORA_OK) return st;
    const int m = n_local_dofs(dim, element);
    const int nv = dim + 1;
    std::map<std::array<int, 3>, int64_t> qid;
    for (int64_t q = 0; q < n_query; ++q) qid[{query[3 * q], query[3 * q + 1], query[3 * q + 2]}] = q;
    std::vector<std::map<std::array<int, 3>, std::pair<double, double>>> rows((size_t)n_query);
    std::vector<double> verts(nv * dim);
    double M[36], K[36];
    int s[6];
    for (int64_t e = 0; e < n_elems; ++e) {
        const int32_t* g = elems + e * nv;
        std::array<int, 3> keys[6];
        int64_t hit[6];
        bool any = false;
        for (int k = 0; k < m; ++k) {
            keys[k] = entity_key(dim, element, g, k);
            auto it = qid.find(keys[k]);
            hit[k] = it == qid.end() ? -1 : it->second;
            any = any || hit[k] >= 0;
        }
        if (!any) continue;
        for (int v = 0; v < nv; ++v)
            for (int c = 0; c < dim; ++c) verts[v * dim + c] = coords[(int64_t)g[v] * dim + c];
        for (int k = 0; k < m; ++k) s[k] = sign_of(dim, element, g, verts.data(), k);
        if (local_matrices(dim, element, verts.data(), s, M, K) != ORA_OK) return ORA_EDEGENERATE;
        for (int k = 0; k < m; ++k) {
            if (hit[k] < 0) continue;
            for (int l = 0; l < m; ++l) {
                auto& a = rows[hit[k]][keys[l]];
                a.first += M[k * m + l];
                a.second += K[k * m + l];
            }
        }
    }
    for (int64_t q = 0; q < n_query; ++q) {
        if ((int)rows[q].size() > cap) return ORA_EINVAL;
        int j = 0;
        for (const auto& kv : rows[q]) {
            for (int c = 0; c < 3; ++c) cols[(q * cap + j) * 3 + c] = kv.first[c];
            vals_M[q * cap + j] = kv.second.first;
            vals_K[q * cap + j] = kv.second.second;
            ++j;
        }
        count[q] = j;
    }
    return ORA_OK;
}

}  // extern "C"

namespace {
/* ===========================================================================
 * vectorized integration (Sec. 3.1):
 * quadrature points F_K(xh_i) for all elements, load vectors against the
 * global basis, L2 norms and field errors.  Same per-element loop style.
 * ======================================================================== */

/* Degree-6 rules on the reference element ("integration
 * quadratures for triangles and tetrahedrons from [Du] and [ZhCuLi]"; the
 * norm listing uses intquad(6, dim)).  2D: Dunavant's
 * 12-point rule; 3D: Keast's 24-point rule (reading C7: any exact rule of the
 * order gives the same integral up to rounding).  Barycentric points,
 * weights normalised to 1 and scaled by |K_hat| = 1/2 resp. 1/6.  Pinned by
 * exact integration of all monomials of degree <= 6 (tests). */
int quad6(int dim, double* pts, double* w) {
    int n = 0;
    auto put = [&](double l1, double l2, double l3, double wt) {  // l0 implied
        pts[dim * n + 0] = l1;
        pts[dim * n + 1] = l2;
        if (dim == 3) pts[dim * n + 2] = l3;
        w[n] = wt;
        ++n;
    };
    if (dim == 2) {
        const double W[3] = {0.116786275726379, 0.050844906370207, 0.082851075618374};
        const double a1 = 0.501426509658179, b1 = 0.249286745170910;
        const double a2 = 0.873821971016996, b2 = 0.063089014491502;
        const double c0 = 0.053145049844817, c1 = 0.310352451033784, c2 = 0.636502499121399;
        /* (l0, l1, l2) permutations; the point is (l1, l2) */
        const double s1[3][3] = {{a1, b1, b1}, {b1, a1, b1}, {b1, b1, a1}};
        const double s2[3][3] = {{a2, b2, b2}, {b2, a2, b2}, {b2, b2, a2}};
        for (int i = 0; i < 3; ++i) put(s1[i][1], s1[i][2], 0.0, 0.5 * W[0]);
        for (int i = 0; i < 3; ++i) put(s2[i][1], s2[i][2], 0.0, 0.5 * W[1]);
        const double l[3] = {c0, c1, c2};
        const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        for (int i = 0; i < 6; ++i) put(l[perm[i][1]], l[perm[i][2]], 0.0, 0.5 * W[2]);
        return n;
    }
    const double sixth = 1.0 / 6.0;
    const double A[3] = {0.214602871259151684, 0.0406739585346113397, 0.322337890142275646};
    const double WA[3] = {0.0399227502581679, 0.0100772110553207, 0.0553571815436544};
    for (int c = 0; c < 3; ++c) {
        const double a = A[c], b = 1.0 - 3.0 * a;
        /* (l0..l3) = (b,a,a,a) and its 3 other placements */
        put(a, a, a, sixth * WA[c]);
        put(b, a, a, sixth * WA[c]);
        put(a, b, a, sixth * WA[c]);
        put(a, a, b, sixth * WA[c]);
    }
    const double a = 0.0636610018750175299, b = 0.269672331458315867, c = 0.603005664791649076;
    const double wt = sixth * 0.0482142857142857;
    /* the 12 placements of (a, a, b, c) over (l0, l1, l2, l3) */
    const double v[4] = {a, a, b, c};
    int cnt = 0;
    for (int i0 = 0; i0 < 4; ++i0)
        for (int i1 = 0; i1 < 4; ++i1)
            for (int i2 = 0; i2 < 4; ++i2)
                for (int i3 = 0; i3 < 4; ++i3) {
                    if (i0 == i1 || i0 == i2 || i0 == i3 || i1 == i2 || i1 == i3 || i2 == i3) continue;
                    if (i0 > i1) continue; /* the two a's are interchangeable: keep i0 < i1 */
                    /* slot i0 and i1 get a, i2 gets b, i3 gets c */
                    double lam[4];
                    lam[i0] = v[0];
                    lam[i1] = v[1];
                    lam[i2] = v[2];
                    lam[i3] = v[3];
                    put(lam[1], lam[2], lam[3], wt);
                    ++cnt;
                }
    (void)cnt;
    return n;
}

/* Physical point F_K(xh) = B_K xh + b_K. */
void map_point(int dim, const double* verts, const double B[3][3], const double* xh, double* x) {
    for (int r = 0; r < dim; ++r) {
        double acc = verts[r];
        for (int c = 0; c < dim; ++c) acc += B[r][c] * xh[c];
        x[r] = acc;
    }
}

/* Values of the global basis on element K at xh: phi[k][r] (value) and
 * dphi[k][r] (div: nd=1, 2D curl: nd=1, 3D curl: nd=3), sign data included
 * (PAPER.md:240-245 RT, 291-301 Ned, 323-331 signs):
 *   RT:  s_k / det B  B eta_hat_k,      div  = s_k / det B  div_hat
 *   Ned: s_k B^{-T} eta_hat_k,          curl = s_k / det B  curl_hat (2D),
 *                                              s_k / det B  B curl_hat (3D). */
void global_basis(int dim, int element, const double* xh, const double B[3][3], double det, const int* s,
                  double phi[6][3], double dphi[6][3]) {
    double BiT[3][3];
    inverse_transpose(dim, B, det, BiT);
    const int m = n_local_dofs(dim, element);
    const int nd = (dim == 3 && element == ORA_NED0) ? 3 : 1;
    double val[18], dc[18];
    ref_basis(dim, element, xh, val, dc);
    for (int k = 0; k < m; ++k) {
        for (int r = 0; r < dim; ++r) {
            double acc = 0.0;
            for (int c = 0; c < dim; ++c)
                acc += (element == ORA_RT0 ? B[r][c] : BiT[r][c]) * val[k * dim + c];
            phi[k][r] = element == ORA_RT0 ? s[k] * acc / det : s[k] * acc;
        }
        if (nd == 3) {
            for (int r = 0; r < 3; ++r) {
                double acc = 0.0;
                for (int c = 0; c < 3; ++c) acc += B[r][c] * dc[3 * k + c];
                dphi[k][r] = s[k] * acc / det;
            }
        } else {
            dphi[k][0] = s[k] * dc[k] / det;
        }
    }
}

}  // namespace

extern "C" {

int ora_quad6(int dim, double* pts, double* w) {
    if (dim != 2 && dim != 3) return ORA_EINVAL;
    return quad6(dim, pts, w);
}

/* pts[(e*nq + q)*dim + r] = F_K(xh_q) for every element (degree-6 rule). */
int ora_quad_points(int dim, int64_t n_elems, const double* coords, const int32_t* elems, double* pts) {
    if (dim != 2 && dim != 3) return ORA_EINVAL;
    double xh[72], w[24];
    const int nq = quad6(dim, xh, w), nv = dim + 1;
    std::vector<double> verts(nv * dim);
    for (int64_t e = 0; e < n_elems; ++e) {
        for (int v = 0; v < nv; ++v)
            for (int c = 0; c < dim; ++c) verts[v * dim + c] = coords[(int64_t)elems[e * nv + v] * dim + c];
        double B[3][3];
        affine(dim, verts.data(), B);
        for (int q = 0; q < nq; ++q) map_point(dim, verts.data(), B, xh + dim * q, pts + (e * nq + q) * dim);
    }
    return nq;
}

/* Load vector b_i = sum_K sum_q w_q |det B_K| f(F_K(xh_q)) . phi_i(xh_q)
 * (pairing 0, f a d-vector) or  . (div / curl phi_i)(xh_q) (pairing 1, f
 * with nd components), accumulated in element order.  e2d / signs are the
 * oracle's own (ora_assemble).  fq[(e*nq + q)*nf + c]. */
int ora_load(int dim, int element, int pairing, int64_t n_elems, const double* coords, const int32_t* elems,
             const int32_t* e2d, const int8_t* signs, int64_t n_dofs, const double* fq, double* b) {
    if ((dim != 2 && dim != 3) || (element != ORA_RT0 && element != ORA_NED0)) return ORA_EINVAL;
    double xh[72], w[24];
    const int nq = quad6(dim, xh, w), nv = dim + 1, m = n_local_dofs(dim, element);
    const int nd = (dim == 3 && element == ORA_NED0) ? 3 : 1;
    const int nf = pairing == 0 ? dim : nd;
    for (int64_t i = 0; i < n_dofs; ++i) b[i] = 0.0;
    std::vector<double> verts(nv * dim);
    for (int64_t e = 0; e < n_elems; ++e) {
        for (int v = 0; v < nv; ++v)
            for (int c = 0; c < dim; ++c) verts[v * dim + c] = coords[(int64_t)elems[e * nv + v] * dim + c];
        double B[3][3];
        const double det = affine(dim, verts.data(), B);
        if (!(det != 0.0)) return ORA_EDEGENERATE;
        int s[6];
        for (int k = 0; k < m; ++k) s[k] = signs[e * m + k];
        double loc[6] = {0, 0, 0, 0, 0, 0};
        for (int q = 0; q < nq; ++q) {
            double phi[6][3], dphi[6][3];
            global_basis(dim, element, xh + dim * q, B, det, s, phi, dphi);
            const double* f = fq + (e * nq + q) * nf;
            for (int k = 0; k < m; ++k) {
                double dot = 0.0;
                for (int c = 0; c < nf; ++c) dot += f[c] * (pairing == 0 ? phi[k][c] : dphi[k][c]);
                loc[k] += w[q] * std::fabs(det) * dot;
            }
        }
        for (int k = 0; k < m; ++k) b[e2d[e * m + k]] += loc[k];
    }
    return ORA_OK;
}

/* ||f||^2 = sum_K sum_q w_q |det B_K| |f(F_K(xh_q))|^2 (PAPER.md:633-645,
 * norm_L2 listing); per_elem[e] = ||f||^2_K; *total = their sum in element
 * order. */
int ora_norm_l2(int dim, int64_t n_elems, const double* coords, const int32_t* elems, const double* fq, int nf,
                double* per_elem, double* total) {
    if (dim != 2 && dim != 3) return ORA_EINVAL;
    double xh[72], w[24];
    const int nq = quad6(dim, xh, w), nv = dim + 1;
    std::vector<double> verts(nv * dim);
    double sum = 0.0;
    for (int64_t e = 0; e < n_elems; ++e) {
        for (int v = 0; v < nv; ++v)
            for (int c = 0; c < dim; ++c) verts[v * dim + c] = coords[(int64_t)elems[e * nv + v] * dim + c];
        double B[3][3];
        const double adet = std::fabs(affine(dim, verts.data(), B));
        double acc = 0.0;
        for (int q = 0; q < nq; ++q) {
            const double* f = fq + (e * nq + q) * nf;
            double f2 = 0.0;
            for (int c = 0; c < nf; ++c) f2 += f[c] * f[c];
            acc += w[q] * adet * f2;
        }
        if (per_elem) per_elem[e] = acc;
        sum += acc;
    }
    *total = sum;
    return ORA_OK;
}

/* Error of the discrete field v = sum_i c_i phi_i against exact values at the
 * quadrature points: err[0] = ||E - v||^2, err[1] = ||D E - D v||^2 with
 * D = div (RT) or curl (Ned).  Eq[(e*nq+q)*dim + r], Dq[(e*nq+q)*nd + r]. */
int ora_field_error(int dim, int element, int64_t n_elems, const double* coords, const int32_t* elems,
                    const int32_t* e2d, const int8_t* signs, const double* coeffs, const double* Eq,
                    const double* Dq, double* err) {
    if ((dim != 2 && dim != 3) || (element != ORA_RT0 && element != ORA_NED0)) return ORA_EINVAL;
    double xh[72], w[24];
    const int nq = quad6(dim, xh, w), nv = dim + 1, m = n_local_dofs(dim, element);
    const int nd = (dim == 3 && element == ORA_NED0) ? 3 : 1;
    std::vector<double> verts(nv * dim);
    double ev = 0.0, ed = 0.0;
    for (int64_t e = 0; e < n_elems; ++e) {
        for (int v = 0; v < nv; ++v)
            for (int c = 0; c < dim; ++c) verts[v * dim + c] = coords[(int64_t)elems[e * nv + v] * dim + c];
        double B[3][3];
        const double det = affine(dim, verts.data(), B);
        if (!(det != 0.0)) return ORA_EDEGENERATE;
        int s[6];
        for (int k = 0; k < m; ++k) s[k] = signs[e * m + k];
        for (int q = 0; q < nq; ++q) {
            double phi[6][3], dphi[6][3];
            global_basis(dim, element, xh + dim * q, B, det, s, phi, dphi);
            double v[3] = {0, 0, 0}, dv[3] = {0, 0, 0};
            for (int k = 0; k < m; ++k) {
                const double ck = coeffs[e2d[e * m + k]];
                for (int r = 0; r < dim; ++r) v[r] += ck * phi[k][r];
                for (int r = 0; r < nd; ++r) dv[r] += ck * dphi[k][r];
            }
            double a = 0.0, d = 0.0;
            for (int r = 0; r < dim; ++r) {
                const double t = Eq[(e * nq + q) * dim + r] - v[r];
                a += t * t;
            }
            for (int r = 0; r < nd; ++r) {
                const double t = Dq[(e * nq + q) * nd + r] - dv[r];
                d += t * t;
            }
            ev += w[q] * std::fabs(det) * a;
            ed += w[q] * std::fabs(det) * d;
        }
    }
    err[0] = ev;
    err[1] = ed;
    return ORA_OK;
}

/* ===========================================================================
 * SURVEY.md §8(f) row f3 support: linear nodal (P1) elements, used by the
 * majorant example for the approximation v ("The approximation
 * v was calculated with linear nodal finite elements"; the P1 code is the
 * authors' earlier paper [RaVa]).  Textbook closed forms:
 *   K^K_ab = |K| grad l_a . grad l_b,   M^K_ab = |K| (1 + d_ab) / ((d+1)(d+2)),
 * grad l_i (i >= 1) = row i-1 of B_K^{-1}, grad l_0 = -sum of the others.
 * ======================================================================== */
static void p1_grads(int dim, const double* verts, double gl[4][3], double* vol) {
    double B[3][3];
    const double det = affine(dim, verts, B);
    double BiT[3][3];
    inverse_transpose(dim, B, det, BiT);
    /* B^{-1} row i = column i of B^{-T} */
    for (int i = 0; i < dim; ++i)
        for (int r = 0; r < dim; ++r) gl[i + 1][r] = BiT[r][i];
    for (int r = 0; r < dim; ++r) {
        double s = 0.0;
        for (int i = 1; i <= dim; ++i) s += gl[i][r];
        gl[0][r] = -s;
    }
    *vol = std::fabs(det) / (dim == 2 ? 2.0 : 6.0);
}

void* ora_p1_assemble(int dim, int64_t n_nodes, int64_t n_elems, const double* coords, const int32_t* elems,
                      int* status) {
    *status = validate(dim, ORA_RT0, n_nodes, n_elems, elems);
    if (*status != ORA_OK) return nullptr;
    Result* R = new Result;
    R->dim = dim;
    const int nv = dim + 1;
    std::map<std::pair<int32_t, int32_t>, std::pair<double, double>> acc;
    std::vector<double> verts(nv * dim);
    for (int64_t e = 0; e < n_elems; ++e) {
        const int32_t* g = elems + e * nv;
        for (int v = 0; v < nv; ++v)
            for (int c = 0; c < dim; ++c) verts[v * dim + c] = coords[(int64_t)g[v] * dim + c];
        double gl[4][3], vol;
        p1_grads(dim, verts.data(), gl, &vol);
        if (!(vol > 0.0)) {
            *status = ORA_EDEGENERATE;
            delete R;
            return nullptr;
        }
        for (int a = 0; a < nv; ++a)
            for (int b = 0; b < nv; ++b) {
                double dot = 0.0;
                for (int r = 0; r < dim; ++r) dot += gl[a][r] * gl[b][r];
                auto& x = acc[{g[a], g[b]}];
                x.first += vol * (a == b ? 2.0 : 1.0) / ((dim + 1) * (dim + 2));
                x.second += vol * dot;
            }
    }
    R->row_ptr.assign((size_t)n_nodes + 1, 0);
    for (const auto& kv : acc) {
        R->row_ptr[kv.first.first + 1] += 1;
        R->col_idx.push_back(kv.first.second);
        R->vals_M.push_back(kv.second.first);
        R->vals_K.push_back(kv.second.second);
    }
    for (int64_t r = 0; r < n_nodes; ++r) R->row_ptr[r + 1] += R->row_ptr[r];
    return R;
}

/* b_a = sum_K sum_q w_q |det B_K| f(x_q) l_a(xh_q), degree-6 points. */
int ora_p1_load(int dim, int64_t n_elems, const double* coords, const int32_t* elems, int64_t n_nodes,
                const double* fq, double* b) {
    if (dim != 2 && dim != 3) return ORA_EINVAL;
    double xh[72], w[24];
    const int nq = quad6(dim, xh, w), nv = dim + 1;
    for (int64_t i = 0; i < n_nodes; ++i) b[i] = 0.0;
    std::vector<double> verts(nv * dim);
    for (int64_t e = 0; e < n_elems; ++e) {
        const int32_t* g = elems + e * nv;
        for (int v = 0; v < nv; ++v)
            for (int c = 0; c < dim; ++c) verts[v * dim + c] = coords[(int64_t)g[v] * dim + c];
        double B[3][3];
        const double adet = std::fabs(affine(dim, verts.data(), B));
        for (int q = 0; q < nq; ++q) {
            double lam[4];
            lam[0] = 1.0;
            for (int i = 0; i < dim; ++i) {
                lam[i + 1] = xh[dim * q + i];
                lam[0] -= lam[i + 1];
            }
            const double f = fq[e * nq + q];
            for (int a = 0; a < nv; ++a) b[g[a]] += w[q] * adet * f * lam[a];
        }
    }
    return ORA_OK;
}

/* grad v on every element (piecewise constant): grad[e*dim + r]. */
int ora_p1_grad(int dim, int64_t n_elems, const double* coords, const int32_t* elems, const double* v,
                double* grad) {
    if (dim != 2 && dim != 3) return ORA_EINVAL;
    const int nv = dim + 1;
    std::vector<double> verts(nv * dim);
    for (int64_t e = 0; e < n_elems; ++e) {
        const int32_t* g = elems + e * nv;
        for (int k = 0; k < nv; ++k)
            for (int c = 0; c < dim; ++c) verts[k * dim + c] = coords[(int64_t)g[k] * dim + c];
        double gl[4][3], vol;
        p1_grads(dim, verts.data(), gl, &vol);
        for (int r = 0; r < dim; ++r) {
            double s = 0.0;
            for (int a = 0; a < nv; ++a) s += v[g[a]] * gl[a][r];
            grad[e * dim + r] = s;
        }
    }
    return ORA_OK;
}

}  // extern "C"
