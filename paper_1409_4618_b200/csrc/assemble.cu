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

// Entity of row i inside element g: returns local index k or -1.
template <class KT>
__device__ __forceinline__ int local_index(const int (&g)[KT::NV], int lv, int b, int c) {
    int q = -1, r = -1;
#pragma unroll
    for (int v = 0; v < KT::NV; ++v) {
        if (g[v] == b) q = v;
        if constexpr (KT::FACES) {
            if (g[v] == c) r = v;
        }
    }
    if (q < 0) return -1;
    if constexpr (KT::FACES) {
        if (r < 0) return -1;
        const int o = 6 - lv - q - r;  // vertex opposite the face
        return 3 - o;
    } else if constexpr (KT::D == 2) {
        return 3 - lv - q;  // 2D edge k is opposite vertex k
    } else {
        const int lo = min(lv, q), hi = max(lv, q);
        // {0,1}->0 {0,2}->1 {0,3}->2 {1,2}->3 {2,3}->4 {1,3}->5
        return lo == 0 ? hi - 1 : (hi == 2 ? 3 : (lo == 2 ? 4 : 5));
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
// Row kernels.  Thread per row; TPB rows per CTA.
// ---------------------------------------------------------------------------------
constexpr int ROW_TPB = 128;

template <class KT>
struct RowCaps {
    // expected max nnz per row for the smem staging budget (falls back to
    // direct global writes when a tile's segment does not fit)
    static constexpr int STAGE_PER_ROW = KT::D == 2 ? 6 : (KT::FACES ? 8 : 18);
    static constexpr int STAGE = ROW_TPB * STAGE_PER_ROW;
    static constexpr int SCRATCH_PER_ROW = KT::D == 2 ? 16 : (KT::FACES ? 16 : 48);
};

// Collect the elements containing entity (a,b[,c]) from a's incidence list,
// sorted ascending by element id.  Returns count (or -1 on overflow).
template <class KT>
__device__ __forceinline__ int row_elements(const int32_t* __restrict__ elems, const int32_t* __restrict__ n2e,
                                            int beg, int end, int b, int c, int* el, int* ek) {
    int ne = 0;
    for (int p = beg; p < end; ++p) {
        const int ent = __ldg(n2e + p);
        const int e = ent >> 2, lv = ent & 3;
        int g[KT::NV];
        load_g<KT>(elems, e, g);
        const int k = local_index<KT>(g, lv, b, c);
        if (k < 0) continue;
        if (ne >= EFEM_MAX_ROW_ELEMS) return -1;
        int j = ne;
        while (j > 0 && el[j - 1] > e) {
            el[j] = el[j - 1];
            ek[j] = ek[j - 1];
            --j;
        }
        el[j] = e;
        ek[j] = k;
        ++ne;
    }
    return ne;
}

template <class KT>
__global__ void __launch_bounds__(ROW_TPB) k_row_count(const int32_t* __restrict__ elems,
                                                       const int32_t* __restrict__ n2e_ptr,
                                                       const int32_t* __restrict__ n2e,
                                                       const int32_t* __restrict__ d2n,
                                                       const int32_t* __restrict__ e2d, int64_t n_rows,
                                                       int32_t* __restrict__ row_cnt, WsHeader* hdr) {
    constexpr int SC = RowCaps<KT>::SCRATCH_PER_ROW;
    __shared__ int scratch[ROW_TPB * SC];
    const int64_t i = blockIdx.x * (int64_t)ROW_TPB + threadIdx.x;
    if (i >= n_rows) return;
    const int a = __ldg(d2n + i * KT::EK), b = __ldg(d2n + i * KT::EK + 1);
    const int c = KT::FACES ? __ldg(d2n + i * KT::EK + 2) : -1;
    int el[EFEM_MAX_ROW_ELEMS], ek[EFEM_MAX_ROW_ELEMS];
    const int ne = row_elements<KT>(elems, n2e, __ldg(n2e_ptr + a), __ldg(n2e_ptr + a + 1), b, c, el, ek);
    if (ne < 0) {
        atomicOr(&hdr->flags[F_CAPACITY], 1);
        row_cnt[i] = 0;
        return;
    }
    int* sc = scratch + threadIdx.x;  // strided by ROW_TPB: conflict-free
    int n = 0;
    bool ok = true;
    for (int t = 0; t < ne; ++t) {
        const int32_t* dofs = e2d + (int64_t)el[t] * KT::M;
#pragma unroll
        for (int l = 0; l < KT::M; ++l) {
            const int col = __ldg(dofs + l);
            int j = n;
            while (j > 0 && sc[(j - 1) * ROW_TPB] > col) --j;
            if (j > 0 && sc[(j - 1) * ROW_TPB] == col) continue;
            if (n >= SC) { ok = false; continue; }
            for (int u = n; u > j; --u) sc[u * ROW_TPB] = sc[(u - 1) * ROW_TPB];
            sc[j * ROW_TPB] = col;
            ++n;
        }
    }
    if (!ok) atomicOr(&hdr->flags[F_CAPACITY], 1);
    row_cnt[i] = n;
}

template <class KT>
__global__ void __launch_bounds__(ROW_TPB) k_row_fill(const double* __restrict__ coords,
                                                      const int32_t* __restrict__ elems,
                                                      const int32_t* __restrict__ n2e_ptr,
                                                      const int32_t* __restrict__ n2e,
                                                      const int32_t* __restrict__ d2n,
                                                      const int32_t* __restrict__ e2d,
                                                      const int32_t* __restrict__ row_ptr, int64_t n_rows,
                                                      unsigned forms, int32_t* __restrict__ col_idx,
                                                      double* __restrict__ vals_m, double* __restrict__ vals_k,
                                                      WsHeader* hdr) {
    constexpr int STAGE = RowCaps<KT>::STAGE;
    constexpr int D = KT::D, NV = KT::NV, M = KT::M;
    __shared__ int s_col[STAGE];
    __shared__ double s_vm[STAGE];
    __shared__ double s_vk[STAGE];

    const int64_t r0 = blockIdx.x * (int64_t)ROW_TPB;
    const int64_t r1 = (r0 + ROW_TPB < n_rows) ? r0 + ROW_TPB : n_rows;
    const int seg0 = __ldg(row_ptr + r0);
    const int segn = __ldg(row_ptr + r1) - seg0;
    const bool staged = segn <= STAGE;
    const int64_t i = r0 + threadIdx.x;

    if (i < n_rows) {
        const int a = __ldg(d2n + i * KT::EK), b = __ldg(d2n + i * KT::EK + 1);
        const int c = KT::FACES ? __ldg(d2n + i * KT::EK + 2) : -1;
        const int rbeg = __ldg(row_ptr + i), rlen = __ldg(row_ptr + i + 1) - rbeg;
        int el[EFEM_MAX_ROW_ELEMS], ek[EFEM_MAX_ROW_ELEMS];
        const int ne = row_elements<KT>(elems, n2e, __ldg(n2e_ptr + a), __ldg(n2e_ptr + a + 1), b, c, el, ek);
        int* cols;
        double *vm, *vk;
        if (staged) {
            cols = s_col + (rbeg - seg0);
            vm = s_vm + (rbeg - seg0);
            vk = s_vk + (rbeg - seg0);
        } else {
            cols = col_idx + rbeg;  // slow path: in-place in global memory
            vm = vals_m;
            vk = vals_k;
            vm = vm ? vm + rbeg : nullptr;
            vk = vk ? vk + rbeg : nullptr;
        }
        int n = 0;
        bool ok = ne >= 0;
        for (int t = 0; ok && t < ne; ++t) {
            const int e = el[t];
            int g[NV];
            load_g<KT>(elems, e, g);
            double X[NV][D];
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int cc = 0; cc < D; ++cc) X[v][cc] = __ldg(coords + (int64_t)g[v] * D + cc);
            double Mr[M], Kr[M];
            const double det = local_row<KT>(X, g, ek[t], Mr, Kr);
            if (!(det != 0.0) || !isfinite(det)) {
                atomicOr(&hdr->flags[F_DEGENERATE], 1);
                atomicMin(&hdr->bad_element, (unsigned long long)e);
            }
            const int32_t* dofs = e2d + (int64_t)e * M;
#pragma unroll
            for (int l = 0; l < M; ++l) {
                const int col = __ldg(dofs + l);
                int j = n;
                while (j > 0 && cols[j - 1] > col) --j;
                if (j > 0 && cols[j - 1] == col) {
                    if (vm) vm[j - 1] += Mr[l];
                    if (vk) vk[j - 1] += Kr[l];
                    continue;
                }
                if (n >= rlen) { ok = false; break; }
                for (int u = n; u > j; --u) {
                    cols[u] = cols[u - 1];
                    if (vm) vm[u] = vm[u - 1];
                    if (vk) vk[u] = vk[u - 1];
                }
                cols[j] = col;
                if (vm) vm[j] = Mr[l];
                if (vk) vk[j] = Kr[l];
                ++n;
            }
        }
        if (!ok || n != rlen) atomicOr(&hdr->flags[F_ROW_MISMATCH], 1);
    }
    if (!staged) return;
    __syncthreads();
    // coalesced flush of this tile's CSR segment
    if (forms & EFEM_PATTERN)
        for (int t = threadIdx.x; t < segn; t += ROW_TPB) col_idx[seg0 + t] = s_col[t];
    if (forms & EFEM_MASS)
        for (int t = threadIdx.x; t < segn; t += ROW_TPB) vals_m[seg0 + t] = s_vm[t];
    if (forms & EFEM_STIFF)
        for (int t = threadIdx.x; t < segn; t += ROW_TPB) vals_k[seg0 + t] = s_vk[t];
}

// ---------------------------------------------------------------------------------
template <class KT>
efem_status launch_rows(Plan& p, bool fill, unsigned forms, efem_csr* out, cudaStream_t s) {
    if (p.n_dofs == 0) return EFEM_OK;
    const unsigned grid = grid_for(p.n_dofs, ROW_TPB);
    if (!fill) {
        k_row_count<KT><<<grid, ROW_TPB, 0, s>>>(p.elems, p.n2e_ptr, p.n2e, p.d2n, p.e2d, p.n_dofs, p.row_cnt,
                                                 p.hdr);
    } else {
        k_row_fill<KT><<<grid, ROW_TPB, 0, s>>>(p.coords, p.elems, p.n2e_ptr, p.n2e, p.d2n, p.e2d, p.row_ptr,
                                                p.n_dofs, forms, out->col_idx,
                                                (forms & EFEM_MASS) ? out->vals_mass : nullptr,
                                                (forms & EFEM_STIFF) ? out->vals_stiff : nullptr, p.hdr);
    }
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status launch_rows_any(Plan& p, bool fill, unsigned forms, efem_csr* out, cudaStream_t s) {
    if (p.dim == 2) return p.element == EFEM_RT0 ? launch_rows<Kind<2, EFEM_RT0>>(p, fill, forms, out, s)
                                                 : launch_rows<Kind<2, EFEM_NED0>>(p, fill, forms, out, s);
    return p.element == EFEM_RT0 ? launch_rows<Kind<3, EFEM_RT0>>(p, fill, forms, out, s)
                                 : launch_rows<Kind<3, EFEM_NED0>>(p, fill, forms, out, s);
}

}  // namespace efem
