// element.cuh -- device helpers of the numeric kernels: element loads,
// orientation signs, closed-form local matrix rows, column ordering masks,
// and the generic (any row shape) row assembler.  Product path only.
#pragma once

#include "efem_internal.cuh"

namespace efem {

// 2D local row in the frame rotated so that vertex q0 (the vertex opposite
// the row's edge) comes first: closed form of PAPER.md:344-363 for the
// sign-corrected Piola-mapped RT0 basis (= NE0 in 2D):
//   M_kl = s_k s_l (y_k . y_l + Q) / (2 |det|),  Q = sum_v |y_v|^2 / 12,
//   K_kl = 2 s_k s_l / |det|,   y_v = x_v - centroid.
// Unsigned values of the row: m0 = M_00, v1 = M_01, v2 = M_02 (x1 = q1,
// x2 = q2), ck = 2 / |det|.  One definition for the numeric kernel
// (assemble.cu tri_row) and the ghost triangles of the distributed path
// (dist2d.cu), so both give the same bits.
struct TriVals {
    double det, m0, v1, v2, ck;
};

__device__ __forceinline__ TriVals tri_vals(double2 x0, double2 x1, double2 x2) {
    TriVals V;
    const double ax = x1.x - x0.x, ay = x1.y - x0.y;  // q1 - q0
    const double bx = x2.x - x0.x, by = x2.y - x0.y;  // q2 - q0
    V.det = ax * by - bx * ay;
    const double cx = (ax + bx) * (1.0 / 3.0), cy = (ay + by) * (1.0 / 3.0);
    const double y0x = -cx, y0y = -cy;
    const double y1x = ax - cx, y1y = ay - cy;
    const double y2x = bx - cx, y2y = by - cy;
    const double n0 = y0x * y0x + y0y * y0y;
    const double Q = (n0 + (y1x * y1x + y1y * y1y) + (y2x * y2x + y2y * y2y)) * (1.0 / 12.0);
    const double rad = 1.0 / fabs(V.det);
    const double cm = 0.5 * rad;
    V.ck = 2.0 * rad;
    V.m0 = cm * (n0 + Q);
    V.v1 = cm * ((y0x * y1x + y0y * y1y) + Q);
    V.v2 = cm * ((y0x * y2x + y0y * y2y) + Q);
    return V;
}

template <class KT>
__device__ __forceinline__ void load_g(const int32_t* __restrict__ elems, int e, int (&g)[KT::NV]) {
    if constexpr (KT::NV == 4) {
        const int4 t = __ldg(reinterpret_cast<const int4*>(elems) + e);
        g[0] = t.x; g[1] = t.y; g[2] = t.z; g[3] = t.w;
    } else {
        const int32_t* p = elems + (int64_t)e * 3;
        g[0] = __ldg(p); g[1] = __ldg(p + 1); g[2] = __ldg(p + 2);
    }
}

// orientation signs (see dofs.cu local_sign for the derivation)
template <class KT>
__device__ __forceinline__ double sign_d(const int (&g)[KT::NV], int k) {
    if constexpr (KT::FACES) {
        const int o = 3 - k;
        int f[3], t = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v)
            if (v != o) f[t++] = g[v];
        const int inv = (f[0] > f[1]) + (f[0] > f[2]) + (f[1] > f[2]);
        return ((inv + (k & 1)) & 1) ? 1.0 : -1.0;
    } else {
        return g[edge_start(KT::D, k)] < g[edge_end(KT::D, k)] ? 1.0 : -1.0;
    }
}

// Row k of the local mass and stiffness matrices of one element, including
// the sign data s_k s_l (PAPER.md:344-363 with reading C2).  Closed forms:
//  RT (2D, 3D) and NE (2D): the Piola-mapped local functions are
//    s_k (x - p_k) / (d |K|) * sign(det)   (p_k = vertex opposite DOF k), so
//    M_kl = s_k s_l (y_k . y_l + Q) / (d^2 |K|),  y_a = x_a - centroid,
//    Q = sum_a |y_a|^2 / ((d+1)(d+2));   K_kl = s_k s_l / |K|.
//    (2D NE0 equals 2D RT0 on the same mesh; pinned by the
//    oracle's own quadrature in the parity tests.)
//  NE (3D): Whitney form lambda_i grad lambda_j - lambda_j grad lambda_i of
//    edge i->j; with G_ab = grad lambda_a . grad lambda_b,
//    M_(ij)(pq) = |K|/20 [(1+d_ip) G_jq - (1+d_iq) G_jp - (1+d_jp) G_iq + (1+d_jq) G_ip]
//    K_(ij)(pq) = 4 |K| (G_ip G_jq - G_iq G_jp).
// Returns det B_K (0 -> degenerate).
template <class KT>
__device__ __forceinline__ double local_row(const double (&X)[KT::NV][KT::D], const int (&g)[KT::NV], int k,
                                            double (&Mr)[KT::M], double (&Kr)[KT::M]) {
    constexpr int D = KT::D, NV = KT::NV, M = KT::M;
    double s[M];
#pragma unroll
    for (int l = 0; l < M; ++l) s[l] = sign_d<KT>(g, l);
    double sk = s[0];
#pragma unroll
    for (int l = 1; l < M; ++l) sk = (k == l) ? s[l] : sk;

    double det;
    if constexpr (D == 2) {
        det = (X[1][0] - X[0][0]) * (X[2][1] - X[0][1]) - (X[2][0] - X[0][0]) * (X[1][1] - X[0][1]);
    } else {
        const double e1[3] = {X[1][0] - X[0][0], X[1][1] - X[0][1], X[1][2] - X[0][2]};
        const double e2[3] = {X[2][0] - X[0][0], X[2][1] - X[0][1], X[2][2] - X[0][2]};
        const double e3[3] = {X[3][0] - X[0][0], X[3][1] - X[0][1], X[3][2] - X[0][2]};
        det = e1[0] * (e2[1] * e3[2] - e2[2] * e3[1]) - e1[1] * (e2[0] * e3[2] - e2[2] * e3[0]) +
              e1[2] * (e2[0] * e3[1] - e2[1] * e3[0]);
    }
    const double adet = fabs(det);

    if constexpr (KT::ELEMENT == EFEM_NED0 && D == 3) {
        // gradients of barycentrics: rows of B^{-1} = (e2 x e3, e3 x e1, e1 x e2) / det
        const double e1[3] = {X[1][0] - X[0][0], X[1][1] - X[0][1], X[1][2] - X[0][2]};
        const double e2[3] = {X[2][0] - X[0][0], X[2][1] - X[0][1], X[2][2] - X[0][2]};
        const double e3[3] = {X[3][0] - X[0][0], X[3][1] - X[0][1], X[3][2] - X[0][2]};
        const double rdet = 1.0 / det;
        double gl[4][3];
        gl[1][0] = (e2[1] * e3[2] - e2[2] * e3[1]) * rdet;
        gl[1][1] = (e2[2] * e3[0] - e2[0] * e3[2]) * rdet;
        gl[1][2] = (e2[0] * e3[1] - e2[1] * e3[0]) * rdet;
        gl[2][0] = (e3[1] * e1[2] - e3[2] * e1[1]) * rdet;
        gl[2][1] = (e3[2] * e1[0] - e3[0] * e1[2]) * rdet;
        gl[2][2] = (e3[0] * e1[1] - e3[1] * e1[0]) * rdet;
        gl[3][0] = (e1[1] * e2[2] - e1[2] * e2[1]) * rdet;
        gl[3][1] = (e1[2] * e2[0] - e1[0] * e2[2]) * rdet;
        gl[3][2] = (e1[0] * e2[1] - e1[1] * e2[0]) * rdet;
#pragma unroll
        for (int c = 0; c < 3; ++c) gl[0][c] = -(gl[1][c] + gl[2][c] + gl[3][c]);
        const int i = (k < 3 ? 0 : (k == 3 ? 1 : (k == 4 ? 2 : 3)));
        const int j = k < 3 ? k + 1 : (k == 3 ? 2 : (k == 4 ? 3 : 1));
        double gi[3], gj[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            gi[c] = i == 0 ? gl[0][c] : (i == 1 ? gl[1][c] : (i == 2 ? gl[2][c] : gl[3][c]));
            gj[c] = j == 1 ? gl[1][c] : (j == 2 ? gl[2][c] : (j == 3 ? gl[3][c] : gl[0][c]));
        }
        double A[4], B[4];  // A_p = G_ip, B_p = G_jp
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            A[q] = gi[0] * gl[q][0] + gi[1] * gl[q][1] + gi[2] * gl[q][2];
            B[q] = gj[0] * gl[q][0] + gj[1] * gl[q][1] + gj[2] * gl[q][2];
        }
        const double vol = adet * (1.0 / 6.0);
        const double cm = vol * (1.0 / 20.0), ck = 4.0 * vol;
#pragma unroll
        for (int l = 0; l < 6; ++l) {
            const int p = edge_start(3, l), q = edge_end(3, l);
            const double dip = (i == p) ? 2.0 : 1.0, diq = (i == q) ? 2.0 : 1.0;
            const double djp = (j == p) ? 2.0 : 1.0, djq = (j == q) ? 2.0 : 1.0;
            const double ss = sk * s[l];
            Mr[l] = ss * cm * (dip * B[q] - diq * B[p] - djp * A[q] + djq * A[p]);
            Kr[l] = ss * ck * (A[p] * B[q] - A[q] * B[p]);
        }
    } else {
        // RT0 2D/3D and NE0 2D: y_a = x_a - centroid, formed from the edge
        // vectors x_a - x_0 (exact differences of neighbouring coordinates) so
        // that no O(1) coordinate is rounded at the O(h) scale of y
        double ev[NV][D];
        double cen[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            ev[0][c] = 0.0;
            double acc = 0.0;
#pragma unroll
            for (int v = 1; v < NV; ++v) {
                ev[v][c] = X[v][c] - X[0][c];
                acc += ev[v][c];
            }
            cen[c] = acc * (1.0 / NV);
        }
        double y[NV][D];
        double sq = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int c = 0; c < D; ++c) {
                y[v][c] = ev[v][c] - cen[c];
                sq += y[v][c] * y[v][c];
            }
        const double Q = sq * (1.0 / ((D + 1) * (D + 2)));
        // opposite vertex of DOF l: 2D -> l, 3D faces -> 3 - l
        const int ok_ = KT::FACES ? 3 - k : k;
        double yk[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double t = y[0][c];
#pragma unroll
            for (int v = 1; v < NV; ++v) t = (ok_ == v) ? y[v][c] : t;
            yk[c] = t;
        }
        // |K| = |det| / d!;  M scale 1/(d^2 |K|) = (d!/d^2)/|det|;  K scale 1/|K| = d!/|det|
        const double rad = 1.0 / adet;
        const double cm = (D == 2 ? 0.5 : 2.0 / 3.0) * rad;
        const double ck = (D == 2 ? 2.0 : 6.0) * rad;
#pragma unroll
        for (int l = 0; l < M; ++l) {
            const int ol = KT::FACES ? 3 - l : l;
            double dot = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) dot += yk[c] * y[ol][c];
            const double ss = sk * s[l];
            Mr[l] = ss * cm * (dot + Q);
            Kr[l] = ss * ck;
        }
    }
    return det;
}

// ---------------------------------------------------------------------------------
// Column order without sorting (row_generic): every column of row i is an
// entity whose nodes lie in W = the sorted set of vertices of the elements
// containing entity i.  DOF ids are lexicographic in node ids and W is sorted
// by node id, so the column order equals the lexicographic order of the
// entities' position tuples in W.  Each present column sets one bit of a
// 256-bit mask at its lexicographic pair / triple index; its CSR slot is the
// popcount of the mask below that bit.
// ---------------------------------------------------------------------------------
constexpr int ROW_TPB = 128;
constexpr int WCAP_EDGE = 23;  // C(23, 2) = 253 <= 256 mask bits
constexpr int WCAP_FACE = 6;   // 6^3 = 216 <= 256

template <class KT>
struct RowCaps {
    // smem staging budget per row (a tile that does not fit writes directly
    // to global memory -- slower, same result)
    static constexpr int STAGE_PER_ROW = KT::D == 2 ? 6 : (KT::FACES ? 8 : 18);
    static constexpr int STAGE = ROW_TPB * STAGE_PER_ROW;
    static constexpr int WCAP = KT::FACES ? WCAP_FACE : WCAP_EDGE;
};

// lexicographic index of local entity l of an element whose vertex positions
// in W are pos[0..NV)
template <class KT>
__device__ __forceinline__ int entity_index(const int (&pos)[KT::NV], int l, int nw) {
    if constexpr (KT::FACES) {
        const int o = 3 - l;
        int f[3], t = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v)
            if (v != o) f[t++] = pos[v];
        const int lo = min(f[0], min(f[1], f[2])), hi = max(f[0], max(f[1], f[2]));
        const int mid = f[0] + f[1] + f[2] - lo - hi;
        return (lo * WCAP_FACE + mid) * WCAP_FACE + hi;
    } else {
        const int u = pos[edge_start(KT::D, l)], v = pos[edge_end(KT::D, l)];
        const int p = min(u, v), q = max(u, v);
        return p * nw - ((p * (p + 1)) >> 1) + (q - p - 1);
    }
}

struct Mask256 {
    unsigned long long w[4];
    int pc[4];
    __device__ __forceinline__ void clear() { w[0] = w[1] = w[2] = w[3] = 0ull; }
    __device__ __forceinline__ void set(int idx) {
        const unsigned long long b = 1ull << (idx & 63);
        const int q = idx >> 6;
        w[0] |= q == 0 ? b : 0ull;
        w[1] |= q == 1 ? b : 0ull;
        w[2] |= q == 2 ? b : 0ull;
        w[3] |= q == 3 ? b : 0ull;
    }
    __device__ __forceinline__ int finish() {
        pc[0] = 0;
        pc[1] = __popcll(w[0]);
        pc[2] = pc[1] + __popcll(w[1]);
        pc[3] = pc[2] + __popcll(w[2]);
        return pc[3] + __popcll(w[3]);
    }
    __device__ __forceinline__ int rank(int idx) const {
        const int q = idx >> 6;
        const unsigned long long word = q == 0 ? w[0] : (q == 1 ? w[1] : (q == 2 ? w[2] : w[3]));
        const int base = q == 0 ? pc[0] : (q == 1 ? pc[1] : (q == 2 ? pc[2] : pc[3]));
        return base + __popcll(word & ((1ull << (idx & 63)) - 1ull));
    }
};


// Generic row: any t <= EFEM_MAX_ROW_ELEMS, |W| <= WCAP.  Accumulates into
// cols / vm / vk (shared staging or global), returns false on a capacity or
// row-length mismatch.
template <class KT>
__device__ __noinline__ bool row_generic(const double* __restrict__ coords, const int32_t* __restrict__ elems,
                                         const int32_t* __restrict__ inc, const int32_t* __restrict__ e2d, int ib,
                                         int t, int rlen, int* cols, double* vm, double* vk, int st,
                                         WsHeader* hdr) {
    constexpr int WCAP = RowCaps<KT>::WCAP;
    constexpr int D = KT::D, NV = KT::NV, M = KT::M;
    bool ok = t <= EFEM_MAX_ROW_ELEMS;
    bool cap = !ok;  // a per-thread capacity (not a mesh defect): reported as EFEM_ECAPACITY
    const int nt = ok ? t : EFEM_MAX_ROW_ELEMS;
    // the row's instances in ascending element order (fixed summation order)
    int ord[EFEM_MAX_ROW_ELEMS];
    for (int j = 0; j < nt; ++j) {
        const int v = __ldg(inc + ib + j) & INST_MASK;
        int q = j;
        while (q > 0 && ord[q - 1] > v) {
            ord[q] = ord[q - 1];
            --q;
        }
        ord[q] = v;
    }
    // pass 1: W = sorted distinct vertices of the row's elements
    int W[WCAP + 1];
    int nw = 0;
    for (int j = 0; j < nt; ++j) {
        const int e = ord[j] >> 3;
        int g[NV];
        load_g<KT>(elems, e, g);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int x = g[v];
            int q = nw;
            while (q > 0 && W[q - 1] > x) --q;
            if (q > 0 && W[q - 1] == x) continue;
            if (nw >= WCAP) { ok = false; cap = true; continue; }
            for (int u = nw; u > q; --u) W[u] = W[u - 1];
            W[q] = x;
            ++nw;
        }
    }
    // pass 2: column mask
    Mask256 mk;
    mk.clear();
    int pk[EFEM_MAX_ROW_ELEMS];
    for (int j = 0; j < nt; ++j) {
        const int e = ord[j] >> 3;
        int g[NV];
        load_g<KT>(elems, e, g);
        int pos[NV];
        int packed = 0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            int lo = 0, hi = nw;  // first index with W >= g[v]
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (W[mid] < g[v]) lo = mid + 1; else hi = mid;
            }
            pos[v] = lo;
            packed |= lo << (5 * v);
        }
        pk[j] = packed;
#pragma unroll
        for (int l = 0; l < M; ++l) mk.set(entity_index<KT>(pos, l, nw));
    }
    const int ncol = mk.finish();
    ok &= ncol == rlen;
    if (cap) atomicOr(&hdr->flags[F_CAPACITY], 1);
    if (!ok) return false;
    for (int q = 0; q < rlen; ++q) {
        vm[q * st] = 0.0;
        vk[q * st] = 0.0;
    }
    // pass 3: values, ascending element id (the incidence list order)
    for (int j = 0; j < nt; ++j) {
        const int pe = ord[j];
        const int e = pe >> 3, k = pe & 7;
        int g[NV];
        load_g<KT>(elems, e, g);
        double X[NV][D];
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int cc = 0; cc < D; ++cc) X[v][cc] = __ldg(coords + (int64_t)g[v] * D + cc);
        int dofs[M];
#pragma unroll
        for (int l = 0; l < M; ++l) dofs[l] = __ldg(e2d + (int64_t)e * M + l);
        double Mr[M], Kr[M];
        const double det = local_row<KT>(X, g, k, Mr, Kr);
        if (!(det != 0.0) || !isfinite(det)) {
            atomicOr(&hdr->flags[F_DEGENERATE], 1);
            atomicMin(&hdr->bad_element, (unsigned long long)e);
        }
        int pos[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) pos[v] = (pk[j] >> (5 * v)) & 31;
#pragma unroll
        for (int l = 0; l < M; ++l) {
            const int slot = mk.rank(entity_index<KT>(pos, l, nw));
            cols[slot * st] = dofs[l];
            vm[slot * st] += Mr[l];
            vk[slot * st] += Kr[l];
        }
    }
    return true;
}

__device__ __forceinline__ int sel4(const int (&g)[4], int i) {
    return i == 0 ? g[0] : (i == 1 ? g[1] : (i == 2 ? g[2] : g[3]));
}


}  // namespace efem
