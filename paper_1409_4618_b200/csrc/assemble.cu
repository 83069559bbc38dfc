// assemble.cu -- sparsity pattern (symbolic) and values (numeric) of the
// global mass / stiffness matrices.
//
// Row-owner design: one thread per global DOF row i.
// The elements containing entity i are found in the incidence list of its
// minimum node; row i's pattern is the union of their elems2dofs rows and its
// values are row k (= local index of entity i) of their local matrices,
// summed in ascending element order.  A CTA stages its rows' CSR segment in
// shared memory and writes it out with coalesced stores, so every CSR byte
// is written exactly once and no T*m^2 contribution array ever reaches HBM.
//
// Local matrices use closed forms of the paper's integrals (DESIGN.md
// "Element math"); the oracle evaluates the same integrals by quadrature.
#include <cub/cub.cuh>

#include "efem_internal.cuh"

namespace efem {

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
        // RT0 2D/3D and NE0 2D: y_a = x_a - centroid
        double cen[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int v = 0; v < NV; ++v) acc += X[v][c];
            cen[c] = acc * (1.0 / NV);
        }
        double y[NV][D];
        double sq = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int c = 0; c < D; ++c) {
                y[v][c] = X[v][c] - cen[c];
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
// Numeric kernel.  Thread per row; ROW_TPB rows per CTA.
//
// Slot of a contribution without sorting: every column of row i is an entity
// whose nodes lie in W = the sorted set of vertices of the elements containing
// entity i (|W| <= 2 + t in 2D, 3 + t for faces, 2 + 2t for 3D edges).
// Since DOF ids are lexicographic in node ids, and W is sorted by node id,
// the column order equals the lexicographic order of the entities' position
// tuples in W.  Each present column sets one bit of a 256-bit mask at its
// lexicographic pair / triple index; its CSR slot is the popcount of the mask
// below that bit.
// ---------------------------------------------------------------------------------
constexpr int ROW_TPB = 128;
constexpr int NE3_SLOTS = 20;  // staged row length cap of the NE0 3D kernel
constexpr size_t NE3_SMEM = (size_t)NE3_SLOTS * ROW_TPB * (8 + 8 + 4) + (ROW_TPB + 1) * 4 + 16 * ROW_TPB;
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


// Coalesced, vectorised copy of a CTA's staged CSR segment to global memory.
// The staging buffers hold element x of the segment at src[sh + x] where
// sh = seg0 mod W, so global and shared addresses have the same alignment
// mod W and the body moves W elements per 16-byte access.
template <class T, class V, int W, int TPB>
__device__ __forceinline__ void flush_vec(T* __restrict__ dst, const T* src, int sh, int n) {
    int head = (W - sh) % W;
    head = head < n ? head : n;
    for (int x = threadIdx.x; x < head; x += TPB) dst[x] = src[sh + x];
    const int nv = (n - head) / W;
    V* dv = reinterpret_cast<V*>(dst + head);
    const V* sv = reinterpret_cast<const V*>(src + sh + head);
    for (int v = threadIdx.x; v < nv; v += TPB) dv[v] = sv[v];
    for (int x = head + nv * W + threadIdx.x; x < n; x += TPB) dst[x] = src[sh + x];
}

__device__ __forceinline__ void flush_segment(unsigned forms, int seg0, int segn, const int* s_col,
                                              const double* s_vm, const double* s_vk, int32_t* col_idx,
                                              double* vals_m, double* vals_k) {
    if (forms & EFEM_PATTERN) flush_vec<int, int4, 4, 128>(col_idx + seg0, s_col, seg0 & 3, segn);
    if (forms & EFEM_MASS) flush_vec<double, double2, 2, 128>(vals_m + seg0, s_vm, seg0 & 1, segn);
    if (forms & EFEM_STIFF) flush_vec<double, double2, 2, 128>(vals_k + seg0, s_vk, seg0 & 1, segn);
}

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
    const int nt = ok ? t : EFEM_MAX_ROW_ELEMS;
    // pass 1: W = sorted distinct vertices of the row's elements
    int W[WCAP + 1];
    int nw = 0;
    for (int j = 0; j < nt; ++j) {
        const int e = __ldg(inc + ib + j) >> 3;
        int g[NV];
        load_g<KT>(elems, e, g);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int x = g[v];
            int q = nw;
            while (q > 0 && W[q - 1] > x) --q;
            if (q > 0 && W[q - 1] == x) continue;
            if (nw >= WCAP) { ok = false; continue; }
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
        const int e = __ldg(inc + ib + j) >> 3;
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
    if (!ok) return false;
    for (int q = 0; q < rlen; ++q) {
        vm[q * st] = 0.0;
        vk[q * st] = 0.0;
    }
    // pass 3: values, ascending element id (the incidence list order)
    for (int j = 0; j < nt; ++j) {
        const int pe = __ldg(inc + ib + j);
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

// 3D edges (NE0).  Row (a, b) with t tets around the edge: the columns are
// the edges among W = {a, b} U link vertices.  Fast path (t <= 7, node ids
// < 2^27): W comes from one 16-key bitonic network in registers
// (key = node << 5 | source), positions go through a per-thread shared
// scratch, the column mask / ranks are as in row_generic.  Other rows use
// row_generic.
template <class KT>
__global__ void __launch_bounds__(ROW_TPB) k_row_fill_ne3(const double* __restrict__ coords,
                                                          const int32_t* __restrict__ elems,
                                                          const int32_t* __restrict__ inc_ptr,
                                                          const int32_t* __restrict__ inc,
                                                          const int32_t* __restrict__ e2d,
                                                          const int32_t* __restrict__ row_ptr, int64_t n_rows,
                                                          unsigned forms, int fast_ids, int32_t* __restrict__ col_idx,
                                                          double* __restrict__ vals_m, double* __restrict__ vals_k,
                                                          WsHeader* hdr) {
    static_assert(KT::D == 3 && !KT::FACES, "NE0 3D only");
    constexpr int TMAX = 7;
    // column-major per-thread accumulators (slot q of row tid at [q * ROW_TPB +
    // tid]: conflict-free), flushed in CSR order through the row offset table
    extern __shared__ __align__(16) unsigned char ne3_smem[];
    double* s_vm = reinterpret_cast<double*>(ne3_smem);
    double* s_vk = s_vm + NE3_SLOTS * ROW_TPB;
    int* s_col = reinterpret_cast<int*>(s_vk + NE3_SLOTS * ROW_TPB);
    int* s_off = s_col + NE3_SLOTS * ROW_TPB;
    unsigned char* s_pos = reinterpret_cast<unsigned char*>(s_off + ROW_TPB + 1);

    const int64_t r0 = blockIdx.x * (int64_t)ROW_TPB;
    const int64_t r1 = (r0 + ROW_TPB < n_rows) ? r0 + ROW_TPB : n_rows;
    const int seg0 = __ldg(row_ptr + r0);
    const int segn = __ldg(row_ptr + r1) - seg0;
    const int64_t i = r0 + threadIdx.x;
    int rbeg = 0, rlen = 0;
    if (i < n_rows) {
        rbeg = __ldg(row_ptr + i);
        rlen = __ldg(row_ptr + i + 1) - rbeg;
        s_off[threadIdx.x] = rbeg - seg0;
    }
    const bool staged = __syncthreads_and(rlen <= NE3_SLOTS);

    if (i < n_rows) {
        const int ib = __ldg(inc_ptr + i);
        const int t = __ldg(inc_ptr + i + 1) - ib;
        int* cols;
        double *vm, *vk;
        int st;
        if (staged) {
            cols = s_col + threadIdx.x;
            vm = s_vm + threadIdx.x;
            vk = s_vk + threadIdx.x;
            st = ROW_TPB;
        } else {
            cols = col_idx + rbeg;  // slow path: accumulate in place in global memory
            vm = vals_m ? vals_m + rbeg : s_vm + threadIdx.x;
            vk = vals_k ? vals_k + rbeg : s_vk + threadIdx.x;
            st = 1;
        }
        bool ok;
        if (fast_ids && t >= 1 && t <= TMAX) {
            unsigned char* P = s_pos + threadIdx.x;  // P[src * ROW_TPB]
            uint32_t key[16];
            int inst[TMAX], roles[TMAX];
            int a = 0, b = 0;
#pragma unroll
            for (int j = 0; j < TMAX; ++j) {
                if (j < t) {
                    const int pe = __ldg(inc + ib + j);
                    inst[j] = pe;
                    const int k = pe & 7;
                    int g[4];
                    load_g<KT>(elems, pe >> 3, g);
                    const int s0 = k < 3 ? 0 : (k == 3 ? 1 : (k == 4 ? 2 : 3));
                    const int s1 = k < 3 ? k + 1 : (k == 3 ? 2 : (k == 4 ? 3 : 1));
                    // complement of {s0, s1}: (2,3) (1,3) (1,2) (0,3) (0,1) (0,2)
                    const int lc = k == 0 ? 2 : (k == 1 ? 1 : (k == 2 ? 1 : 0));
                    const int ld = k == 0 ? 3 : (k == 1 ? 3 : (k == 2 ? 2 : (k == 3 ? 3 : (k == 4 ? 1 : 2))));
                    const int g0 = sel4(g, s0), g1 = sel4(g, s1);
                    const int la = g0 < g1 ? s0 : s1, lb = g0 < g1 ? s1 : s0;
                    a = min(g0, g1);
                    b = max(g0, g1);
                    roles[j] = la | (lb << 2) | (lc << 4) | (ld << 6);
                    key[2 * j] = ((uint32_t)sel4(g, lc) << 5) | (2 * j);
                    key[2 * j + 1] = ((uint32_t)sel4(g, ld) << 5) | (2 * j + 1);
                } else {
                    key[2 * j] = 0xffffffffu;
                    key[2 * j + 1] = 0xffffffffu;
                }
            }
            key[14] = ((uint32_t)a << 5) | 14u;
            key[15] = ((uint32_t)b << 5) | 15u;
            // bitonic sort of 16 keys
#pragma unroll
            for (int kk = 2; kk <= 16; kk <<= 1)
#pragma unroll
                for (int jj = kk >> 1; jj > 0; jj >>= 1)
#pragma unroll
                    for (int x = 0; x < 16; ++x) {
                        const int y = x ^ jj;
                        if (y > x) {
                            const uint32_t lo = min(key[x], key[y]), hi = max(key[x], key[y]);
                            const bool asc = (x & kk) == 0;
                            key[x] = asc ? lo : hi;
                            key[y] = asc ? hi : lo;
                        }
                    }
            // distinct ranks -> positions per source
            int r = -1;
            uint32_t prev = 0xffffffffu;
#pragma unroll
            for (int x = 0; x < 16; ++x) {
                if (key[x] != 0xffffffffu) {
                    const uint32_t v = key[x] >> 5;
                    r += v != prev;
                    prev = v;
                    P[(key[x] & 31u) * ROW_TPB] = (unsigned char)r;
                }
            }
            const int nw = r + 1;
            const int pa = P[14 * ROW_TPB], pb = P[15 * ROW_TPB];
            Mask256 mk;
            mk.clear();
            int pk[TMAX];
#pragma unroll
            for (int j = 0; j < TMAX; ++j) {
                if (j < t) {
                    const int pc = P[(2 * j) * ROW_TPB], pd = P[(2 * j + 1) * ROW_TPB];
                    const int rl = roles[j];
                    int pos[4];
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        pos[v] = v == (rl & 3) ? pa : (v == ((rl >> 2) & 3) ? pb : (v == ((rl >> 4) & 3) ? pc : pd));
                    pk[j] = pos[0] | (pos[1] << 5) | (pos[2] << 10) | (pos[3] << 15);
#pragma unroll
                    for (int l = 0; l < 6; ++l) mk.set(entity_index<KT>(pos, l, nw));
                }
            }
            ok = mk.finish() == rlen;
            if (ok) {
                for (int q = 0; q < rlen; ++q) {
                    vm[q * st] = 0.0;
                    vk[q * st] = 0.0;
                }
#pragma unroll
                for (int j = 0; j < TMAX; ++j) {
                    if (j < t) {
                        const int e = inst[j] >> 3, k = inst[j] & 7;
                        int g[4];
                        load_g<KT>(elems, e, g);
                        double X[4][3];
#pragma unroll
                        for (int v = 0; v < 4; ++v)
#pragma unroll
                            for (int cc = 0; cc < 3; ++cc) X[v][cc] = __ldg(coords + (int64_t)g[v] * 3 + cc);
                        const int2* dp = reinterpret_cast<const int2*>(e2d + (int64_t)e * 6);
                        const int2 d01 = __ldg(dp), d23 = __ldg(dp + 1), d45 = __ldg(dp + 2);
                        const int dofs[6] = {d01.x, d01.y, d23.x, d23.y, d45.x, d45.y};
                        double Mr[6], Kr[6];
                        const double det = local_row<KT>(X, g, k, Mr, Kr);
                        if (!(det != 0.0) || !isfinite(det)) {
                            atomicOr(&hdr->flags[F_DEGENERATE], 1);
                            atomicMin(&hdr->bad_element, (unsigned long long)e);
                        }
                        int pos[4];
#pragma unroll
                        for (int v = 0; v < 4; ++v) pos[v] = (pk[j] >> (5 * v)) & 31;
#pragma unroll
                        for (int l = 0; l < 6; ++l) {
                            const int slot = mk.rank(entity_index<KT>(pos, l, nw));
                            cols[slot * st] = dofs[l];
                            vm[slot * st] += Mr[l];
                            vk[slot * st] += Kr[l];
                        }
                    }
                }
            }
        } else {
            ok = row_generic<KT>(coords, elems, inc, e2d, ib, t, rlen, cols, vm, vk, st, hdr);
        }
        if (!ok) atomicOr(&hdr->flags[F_ROW_MISMATCH], 1);
    }
    if (!staged) return;
    __syncthreads();
    // CSR-order flush: element x of the segment belongs to the last row r with
    // s_off[r] <= x, slot x - s_off[r]
    const int nr = (int)(r1 - r0);
    for (int x = threadIdx.x; x < segn; x += ROW_TPB) {
        int lo = 0, hi = nr - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_off[mid] <= x) lo = mid; else hi = mid - 1;
        }
        const int src = (x - s_off[lo]) * ROW_TPB + lo;
        if (forms & EFEM_PATTERN) col_idx[seg0 + x] = s_col[src];
        if (forms & EFEM_MASS) vals_m[seg0 + x] = s_vm[src];
        if (forms & EFEM_STIFF) vals_k[seg0 + x] = s_vk[src];
    }
}

// ---------------------------------------------------------------------------------
// 2D edges and 3D faces: an entity lies in t <= 2 elements of a conforming
// mesh and its row is {own DOF} + the (m-1) other DOFs of each element, all
// distinct (two elements share at most this entity).  So a row has
// 1 + (m-1) t <= 5 (2D) or 7 (3D faces) entries: gather them in registers,
// sum the own entry over the elements (ascending element id), and order the
// columns with a fixed odd-even transposition network.  No search, no merge.
// ---------------------------------------------------------------------------------
template <class KT>
__global__ void __launch_bounds__(ROW_TPB) k_row_fill_net(const double* __restrict__ coords,
                                                          const int32_t* __restrict__ elems,
                                                          const int32_t* __restrict__ inc_ptr,
                                                          const int32_t* __restrict__ inc,
                                                          const int32_t* __restrict__ e2d,
                                                          const int32_t* __restrict__ row_ptr, int64_t n_rows,
                                                          unsigned forms, int32_t* __restrict__ col_idx,
                                                          double* __restrict__ vals_m, double* __restrict__ vals_k,
                                                          WsHeader* hdr) {
    constexpr int D = KT::D, NV = KT::NV, M = KT::M;
    constexpr int NS = 1 + 2 * (M - 1);
    constexpr int STAGE = ROW_TPB * NS;
    __shared__ __align__(16) int s_col[STAGE + 4];
    __shared__ __align__(16) double s_vm[STAGE + 2];
    __shared__ __align__(16) double s_vk[STAGE + 2];

    const int64_t r0 = blockIdx.x * (int64_t)ROW_TPB;
    const int64_t r1 = (r0 + ROW_TPB < n_rows) ? r0 + ROW_TPB : n_rows;
    const int seg0 = __ldg(row_ptr + r0);
    const int segn = __ldg(row_ptr + r1) - seg0;
    const int64_t i = r0 + threadIdx.x;

    if (i < n_rows) {
        const int ib = __ldg(inc_ptr + i);
        const int t = __ldg(inc_ptr + i + 1) - ib;
        const int rbeg = __ldg(row_ptr + i);
        const int rlen = __ldg(row_ptr + i + 1) - rbeg;
        if (t < 1 || t > 2 || rlen != 1 + (M - 1) * t) {
            atomicOr(&hdr->flags[F_ROW_MISMATCH], 1);
        } else {
            int cols[NS];
            double vm[NS], vk[NS];
            cols[0] = (int)i;
            vm[0] = 0.0;
            vk[0] = 0.0;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (j < t) {
                    const int pe = __ldg(inc + ib + j);
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
                    double om = Mr[0], ok = Kr[0];
#pragma unroll
                    for (int l = 1; l < M; ++l) {
                        om = (k == l) ? Mr[l] : om;
                        ok = (k == l) ? Kr[l] : ok;
                    }
                    vm[0] += om;
                    vk[0] += ok;
#pragma unroll
                    for (int q = 0; q < M - 1; ++q) {  // the other local DOFs, l = q + (q >= k)
                        int c = dofs[q];
                        double a = Mr[q], b = Kr[q];
#pragma unroll
                        for (int l = q + 1; l <= q + 1 && l < M; ++l) {
                            c = (q >= k) ? dofs[l] : c;
                            a = (q >= k) ? Mr[l] : a;
                            b = (q >= k) ? Kr[l] : b;
                        }
                        cols[1 + j * (M - 1) + q] = c;
                        vm[1 + j * (M - 1) + q] = a;
                        vk[1 + j * (M - 1) + q] = b;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < M - 1; ++q) {
                        cols[1 + j * (M - 1) + q] = INT_MAX;
                        vm[1 + j * (M - 1) + q] = 0.0;
                        vk[1 + j * (M - 1) + q] = 0.0;
                    }
                }
            }
            // place by rank: the valid columns are distinct, sentinels (INT_MAX)
            // rank last and are not written
            const int o = rbeg - seg0;
#pragma unroll
            for (int x = 0; x < NS; ++x) {
                int r = 0;
#pragma unroll
                for (int y = 0; y < NS; ++y) r += (y != x) & (cols[y] < cols[x]);
                if (cols[x] != INT_MAX) {
                    s_col[(seg0 & 3) + o + r] = cols[x];
                    s_vm[(seg0 & 1) + o + r] = vm[x];
                    s_vk[(seg0 & 1) + o + r] = vk[x];
                }
            }
        }
    }
    __syncthreads();
    flush_segment(forms, seg0, segn, s_col, s_vm, s_vk, col_idx, vals_m, vals_k);
}

// ---------------------------------------------------------------------------------
template <class KT>
efem_status launch_rows(Plan& p, unsigned forms, efem_csr* out, cudaStream_t s) {
    if (p.n_dofs == 0) return EFEM_OK;
    const unsigned grid = grid_for(p.n_dofs, ROW_TPB);
    double* vm = (forms & EFEM_MASS) ? out->vals_mass : nullptr;
    double* vk = (forms & EFEM_STIFF) ? out->vals_stiff : nullptr;
    if constexpr (KT::D == 2 || KT::FACES) {
        k_row_fill_net<KT><<<grid, ROW_TPB, 0, s>>>(p.coords, p.elems, p.inc_ptr, p.bucket, p.e2d, p.row_ptr,
                                                    p.n_dofs, forms, out->col_idx, vm, vk, p.hdr);
    } else {
        const int fast_ids = p.n_nodes < (1ll << 27);
        static bool attr = false;
        if (!attr) {
            EFEM_CUDA_TRY(cudaFuncSetAttribute(k_row_fill_ne3<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)NE3_SMEM));
            attr = true;
        }
        k_row_fill_ne3<KT><<<grid, ROW_TPB, NE3_SMEM, s>>>(p.coords, p.elems, p.inc_ptr, p.bucket, p.e2d, p.row_ptr,
                                                    p.n_dofs, forms, fast_ids, out->col_idx, vm, vk, p.hdr);
    }
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status launch_rows_any(Plan& p, unsigned forms, efem_csr* out, cudaStream_t s) {
    if (p.dim == 2) return p.element == EFEM_RT0 ? launch_rows<Kind<2, EFEM_RT0>>(p, forms, out, s)
                                                 : launch_rows<Kind<2, EFEM_NED0>>(p, forms, out, s);
    return p.element == EFEM_RT0 ? launch_rows<Kind<3, EFEM_RT0>>(p, forms, out, s)
                                 : launch_rows<Kind<3, EFEM_NED0>>(p, forms, out, s);
}

}  // namespace efem
