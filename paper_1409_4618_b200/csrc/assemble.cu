// assemble.cu -- numeric assembly: local matrices summed
// into the CSR rows of the global mass / stiffness matrices (PAPER.md:335-342,
// 671-696).
//
// Row-owner design: one thread per global DOF row i.  The
// elements containing entity i are the run of the incidence (sorted bucket)
// [inc_ptr[i], inc_ptr[i+1]); row i's values are row k (local index of
// entity i) of their local matrices, summed in ascending element order.
// Rows are staged in shared memory (per warp: k_rows_tri; per CTA:
// k_rows_ne3) and written out with coalesced stores, so every CSR byte is
// written exactly once and no local matrix ever reaches HBM.
#include <atomic>
#include <type_traits>

#include "element.cuh"

namespace efem {

#ifndef EFEM_NE3_WARPFLUSH
#define EFEM_NE3_WARPFLUSH 1
#endif
#ifndef EFEM_NE3_TPB
#define EFEM_NE3_TPB 128
#endif
constexpr int NUM_TPB = EFEM_NE3_TPB;
constexpr int kMaxDevices = 64;

// ---------------------------------------------------------------------------------
// 2D edges and 3D faces.  In a conforming mesh an entity lies in t <= 2
// elements and two elements share at most that entity, so row i is
// {i} U (the m-1 other DOFs of each element): 1 + (m-1) t <= 5 (2D) or 7
// entries, all distinct, and row i starts at i + (m-1) inc_ptr[i] (closed
// form; this kernel also writes row_ptr).  One thread per row; each warp
// stages its 32 rows' CSR segment in shared memory (no block barrier) and
// flushes it with coalesced stores, so every CSR byte is written once.
// ---------------------------------------------------------------------------------

// 2D: local row k of one triangle in the frame rotated so that vertex k (the
// vertex opposite edge k) comes first.  Edge l runs from vertex l+1 to l+2
// (Fig. 1, reading C4), so with q0 = g[k], q1 = g[k+1], q2 = g[k+2]
// the row's edge is q1 -> q2 and the other two are q2 -> q0 (local k+1,
// opposite q1) and q0 -> q1 (local k+2, opposite q2).  Closed form of
// PAPER.md:344-363 (see local_row): M_kl = s_k s_l (y_k.y_l + Q) / (2|det|),
// K_kl = 2 s_k s_l / |det|, y = vertex - centroid, Q = sum |y|^2 / 12.
struct Tri {
    int q0, q1, q2;  // global vertex ids, rotated
    int d1, d2;      // DOF ids of local edges k+1, k+2
    double2 x0, x1, x2;
};

__device__ __forceinline__ int mod3_next(int k) { return k == 2 ? 0 : k + 1; }
__device__ __forceinline__ int mod3_prev(int k) { return k == 0 ? 2 : k - 1; }

__device__ __forceinline__ void tri_load_ids(const int32_t* __restrict__ elems, const int32_t* __restrict__ e2d,
                                             int inst, Tri& T) {
    const int e = inst >> 3, k = inst & 7;
    const int k1 = mod3_next(k), k2 = mod3_prev(k);
    const int32_t* ge = elems + (int64_t)e * 3;
    const int32_t* de = e2d + (int64_t)e * 3;
    T.q0 = __ldg(ge + k);
    T.q1 = __ldg(ge + k1);
    T.q2 = __ldg(ge + k2);
    T.d1 = __ldg(de + k1);
    T.d2 = __ldg(de + k2);
}

__device__ __forceinline__ void tri_load_x(const double* __restrict__ coords, Tri& T) {
    const double2* c2 = reinterpret_cast<const double2*>(coords);
    T.x0 = __ldg(c2 + T.q0);
    T.x1 = __ldg(c2 + T.q1);
    T.x2 = __ldg(c2 + T.q2);
}

// returns det; m0/k0 own entry, m1,k1 / m2,k2 the entries of columns d1, d2
__device__ __forceinline__ double tri_row(const Tri& T, double& m0, double& k0, double& m1, double& k1,
                                          double& m2, double& k2) {
    const TriVals V = tri_vals(T.x0, T.x1, T.x2);
    const bool so = T.q1 < T.q2;  // s_own
    const bool sg1 = so == (T.q2 < T.q0), sg2 = so == (T.q0 < T.q1);  // s_own s_l > 0
    m0 = V.m0;
    k0 = V.ck;
    m1 = sg1 ? V.v1 : -V.v1;
    m2 = sg2 ? V.v2 : -V.v2;
    k1 = sg1 ? V.ck : -V.ck;
    k2 = sg2 ? V.ck : -V.ck;
    return V.det;
}

// Ghost triangles of a distributed assembly (dist2d.cu): triangles of another
// rank's slab whose local matrices that rank computed and sent.  A triangle
// with (local) index e >= base is a ghost; its row k values are
// vals[(e - base) * 12 + 4 k + {0..3}] = {M_kk, M_k,k+1, M_k,k+2 (unsigned), 2/|det|}
// in the same rotated frame tri_row uses (bitwise the values tri_row gives).
// Columns of the distributed path are e2d + col_base (elems2dofs held in
// rank-local ids; the own DOF comes from own_base).
// (GhostArgs: efem_internal.cuh)

// Element policies of the pipelined pair kernel (rows of t <= 2 elements).
// Ids = the gathers that depend only on the instance (L2), Geo = the
// coordinates (L3); row() returns det and fills the own entry and the m-1
// other entries of the element's local row.
struct TriPolicy {
    static constexpr int M = 3;
    static constexpr bool DEEP = true;   // four-stage pipeline, shared-edge loads (load_ids2 / complete2)
    static constexpr bool GHOST = false;
    using Ids = Tri;
    struct Geo {};
    __device__ __forceinline__ static void load_ids(const int32_t* __restrict__ elems,
                                                    const int32_t* __restrict__ e2d, int inst, Ids& I) {
        tri_load_ids(elems, e2d, inst, I);
    }
    __device__ __forceinline__ static void load_x(const double* __restrict__ coords, const GhostArgs&, Ids& I, Geo&) {
        tri_load_x(coords, I);
    }
    __device__ __forceinline__ static double row(const Ids& I, const Geo&, const GhostArgs&, int, double& m0, double& k0,
                                                 int (&c)[2], double (&m)[2], double (&k)[2]) {
        c[0] = I.d1;
        c[1] = I.d2;
        return tri_row(I, m0, k0, m[0], k[0], m[1], k[1]);
    }
    // The row's second triangle shares the row's edge with the first: only
    // its opposite vertex (id + coordinates), its local start vertex (for the
    // orientation) and its two other DOFs are loaded; the rest is taken from
    // the first triangle (13 gathers per interior row instead of 16).
    __device__ __forceinline__ static void load_ids2(const int32_t* __restrict__ elems,
                                                     const int32_t* __restrict__ e2d, int inst, Ids& I) {
        const int e = inst >> 3, k = inst & 7;
        const int k1 = mod3_next(k), k2 = mod3_prev(k);
        const int32_t* ge = elems + (int64_t)e * 3;
        const int32_t* de = e2d + (int64_t)e * 3;
        I.q0 = __ldg(ge + k);
        I.q1 = __ldg(ge + k1);
        I.d1 = __ldg(de + k1);
        I.d2 = __ldg(de + k2);
    }
    __device__ __forceinline__ static void load_x2(const double* __restrict__ coords, Ids& I) {
        I.x0 = __ldg(reinterpret_cast<const double2*>(coords) + I.q0);
    }
    __device__ __forceinline__ static void complete2(const Ids& A, Ids& I) {
        const bool same = I.q1 == A.q1;
        I.q2 = same ? A.q2 : A.q1;
        I.x1 = same ? A.x1 : A.x2;
        I.x2 = same ? A.x2 : A.x1;
    }
};

// 3D faces (RT0).  Face k is the face opposite vertex o = 3 - k; with y_v the
// vertices relative to the centroid, M_kl = s_k s_l (y_o(k).y_o(l) + Q) (2/3)/|det|,
// Q = sum |y|^2 / 20, K_kl = 6 s_k s_l / |det| (see local_row).
struct FacePolicy {
    static constexpr int M = 4;
    static constexpr bool DEEP = false;
    static constexpr bool GHOST = false;
    struct Ids {
        int4 g, d;
        int k;
    };
    struct Geo {
        double x[4][3];
    };
    __device__ __forceinline__ static void load_ids(const int32_t* __restrict__ elems,
                                                    const int32_t* __restrict__ e2d, int inst, Ids& I) {
        const int e = inst >> 3;
        I.k = inst & 7;
        I.g = __ldg(reinterpret_cast<const int4*>(elems) + e);
        I.d = __ldg(reinterpret_cast<const int4*>(e2d) + e);
    }
    __device__ __forceinline__ static void load_x(const double* __restrict__ coords, const GhostArgs&, Ids& I,
                                                  Geo& G) {
        const int g[4] = {I.g.x, I.g.y, I.g.z, I.g.w};
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int c = 0; c < 3; ++c) G.x[v][c] = __ldg(coords + (int64_t)g[v] * 3 + c);
    }
    __device__ __forceinline__ static double row(const Ids& I, const Geo& G, const GhostArgs&, int, double& m0,
                                                 double& k0, int (&c)[3], double (&m)[3], double (&kv)[3]) {
        const int g[4] = {I.g.x, I.g.y, I.g.z, I.g.w};
        const int d[4] = {I.d.x, I.d.y, I.d.z, I.d.w};
        double ev[4][3], cen[3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
            ev[0][cc] = 0.0;
            ev[1][cc] = G.x[1][cc] - G.x[0][cc];
            ev[2][cc] = G.x[2][cc] - G.x[0][cc];
            ev[3][cc] = G.x[3][cc] - G.x[0][cc];
            cen[cc] = (ev[1][cc] + ev[2][cc] + ev[3][cc]) * 0.25;
        }
        const double det = ev[1][0] * (ev[2][1] * ev[3][2] - ev[2][2] * ev[3][1]) -
                           ev[1][1] * (ev[2][0] * ev[3][2] - ev[2][2] * ev[3][0]) +
                           ev[1][2] * (ev[2][0] * ev[3][1] - ev[2][1] * ev[3][0]);
        double y[4][3], sq = 0.0;
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                y[v][cc] = ev[v][cc] - cen[cc];
                sq += y[v][cc] * y[v][cc];
            }
        const double Q = sq * (1.0 / 20.0);
        const double rad = 1.0 / fabs(det);
        const double cm = (2.0 / 3.0) * rad, ck = 6.0 * rad;
        // face signs: s_l = -sgn(ascending face vertices, then the opposite one)
        bool pos[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const int o = 3 - l;
            int f[3], t = 0;
#pragma unroll
            for (int v = 0; v < 4; ++v)
                if (v != o) f[t++] = g[v];
            const int inv = (f[0] > f[1]) + (f[0] > f[2]) + (f[1] > f[2]);
            pos[l] = ((inv + (l & 1)) & 1) != 0;
        }
        const int k = I.k, ok = 3 - k;
        bool sk = pos[0];
        double yo[3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) yo[cc] = y[0][cc];
#pragma unroll
        for (int v = 1; v < 4; ++v) {
            if (ok == v) {
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) yo[cc] = y[v][cc];
            }
            if (k == v) sk = pos[v];
        }
        m0 = cm * ((yo[0] * yo[0] + yo[1] * yo[1] + yo[2] * yo[2]) + Q);
        k0 = ck;
#pragma unroll
        for (int q = 0; q < 3; ++q) {  // the other faces l = q + (q >= k), opposite vertex 3 - l
            const bool sh = q >= k;
            const int l = q + sh;
            const int ol = 3 - l;
            double yl[3];
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                double v = y[0][cc];
#pragma unroll
                for (int w = 1; w < 4; ++w) v = (ol == w) ? y[w][cc] : v;
                yl[cc] = v;
            }
            bool sl = pos[0];
            int dl = d[0];
#pragma unroll
            for (int w = 1; w < 4; ++w) {
                sl = (l == w) ? pos[w] : sl;
                dl = (l == w) ? d[w] : dl;
            }
            const double val = cm * ((yo[0] * yl[0] + yo[1] * yl[1] + yo[2] * yl[2]) + Q);
            const bool same = sk == sl;
            c[q] = dl;
            m[q] = same ? val : -val;
            kv[q] = same ? ck : -ck;
        }
        return det;
    }
};

// 2D with ghost triangles (distributed assembly, dist2d.cu; see above): the
// policy runs on TriPolicy's four-stage pipeline with the shared-edge loads
// (coordinates are loaded for every triangle -- the mesh is whole on every
// rank -- so the second triangle completes from the first); a ghost's values,
// rare (interface rows only), are read when its row is computed.  Columns
// are elems2dofs + col_base.
struct GhostDeepPolicy : TriPolicy {
    static constexpr bool GHOST = true;
    __device__ __forceinline__ static double row(const Ids& I, const Geo&, const GhostArgs& gh, int inst, double& m0,
                                                 double& k0, int (&c)[2], double (&m)[2], double (&k)[2]) {
        c[0] = I.d1 + gh.col_base;
        c[1] = I.d2 + gh.col_base;
        const int e = inst >> 3;
        if (e < gh.base) return tri_row(I, m0, k0, m[0], k[0], m[1], k[1]);
        const double2* v = reinterpret_cast<const double2*>(gh.vals + (int64_t)(e - gh.base) * 12 + 4 * (inst & 7));
        const double2 gv0 = __ldg(v), gv1 = __ldg(v + 1);
        const bool so = I.q1 < I.q2;
        const bool sg1 = so == (I.q2 < I.q0), sg2 = so == (I.q0 < I.q1);
        const double ck = gv1.y;
        m0 = gv0.x;
        k0 = ck;
        m[0] = sg1 ? gv0.y : -gv0.y;
        m[1] = sg2 ? gv1.x : -gv1.x;
        k[0] = sg1 ? ck : -ck;
        k[1] = sg2 ? ck : -ck;
        return 1.0;  // (the sending rank checked the determinant)
    }
};

// 2D, persistent and software-pipelined: every warp walks 32-row batches
// (grid-stride, so concurrently running warps work on neighbouring rows and
// share element data in L2).  The gather chain per row is
//   L1 inc_ptr[i], inc_ptr[i+1], rec[i]  ->  L2 elems / elems2dofs  ->  L3 coords
// and is overlapped across batches: while batch b is computed, the L2 loads
// of batch b+1 and the L1 loads of batch b+2 are in flight.
#ifndef EFEM_TRI_TPB
#define EFEM_TRI_TPB 256
#endif
constexpr int TRI_TPB = EFEM_TRI_TPB;

// Asynchronous assembly (efem_assemble_async): the row count comes from the
// enumeration's header totals on the device; a pattern larger than the output
// capacities is flagged (F_CAPACITY) and nothing is written.  Returns -1 then.
__device__ __forceinline__ int dyn_rows(WsHeader* hdr, int cap_rows, long long cap_nnz) {
    const long long r = *(volatile long long*)&hdr->totals[0], z = *(volatile long long*)&hdr->totals[1];
    if (r > cap_rows || z > cap_nnz) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&hdr->flags[F_CAPACITY], 1);
        return -1;
    }
    return (int)r;
}

// Bound partition (efem_part_numeric_async): rows and entries of the window
// from the device; a window larger than the slice capacities is flagged.
__device__ __forceinline__ int win_rows(WsHeader* hdr, const long long* win, int cap_rows, long long cap_nnz) {
    const long long r = *(volatile const long long*)&win[1], z = *(volatile const long long*)&win[3];
    if (r > cap_rows || z > cap_nnz) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&hdr->flags[F_CAPACITY], 1);
        return -1;
    }
    return (int)r;
}

// L1 of a batch: the lane's row record; lane 0 also the batch's first
// incidence offset (row offsets follow from t = 1 + (first != last) by a
// warp scan, so inc_ptr is read once per batch, not per row)
struct TriL1 {
    int2 rr;
    int ib0;
};

__device__ __forceinline__ TriL1 tri_l1(const int32_t* __restrict__ inc_ptr, const int2* __restrict__ rec, int batch,
                                        int nbatch, int n_rows, int lane) {
    TriL1 a;
    a.ib0 = 0;
    a.rr = make_int2(0, 0);
    if (batch < nbatch) {
        const int li = min(batch * 32 + lane, n_rows - 1);
        a.rr = __ldg(rec + li);
        if (lane == 0) a.ib0 = __ldg(inc_ptr + batch * 32);
    }
    return a;
}

template <class KT, class P, int MINB, bool WIN>
__global__ void __launch_bounds__(TRI_TPB, MINB) k_rows_tri(const double* __restrict__ coords,
                                                           const int32_t* __restrict__ elems,
                                                           const int32_t* __restrict__ inc_ptr,
                                                           const int2* __restrict__ rec,
                                                           const int32_t* __restrict__ e2d, int row0, int n_rows_arg,
                                                           int own_base, int out_base, unsigned forms,
                                                           int32_t* __restrict__ row_ptr_out,
                                                           int32_t* __restrict__ col_idx,
                                                           double* __restrict__ vals_m, double* __restrict__ vals_k,
                                                           WsHeader* hdr, int dyn, long long cap_nnz,
                                                           const long long* __restrict__ win, GhostArgs gh) {
    constexpr int M = P::M, NO = M - 1;
    // node ids out of range (flagged by the enumeration): nothing is gathered
    if (*(volatile const int*)&hdr->flags[F_INVALID_NODE]) return;
    int n_rows = dyn ? dyn_rows(hdr, n_rows_arg, cap_nnz) : n_rows_arg;
    if constexpr (WIN) {  // (a template flag: the common path carries none of this)
        n_rows = win_rows(hdr, win, n_rows_arg, cap_nnz);
        if (n_rows > 0) {
            row0 = (int)win[0];
            out_base = (int)win[2];
            own_base = (int)win[4];
            rec += row0;
            inc_ptr += row0;
            // distributed path: elems2dofs held relative to the rank's first row
            if constexpr (P::GHOST) gh.col_base = own_base;
        }
    }
    if (n_rows <= 0) {
        if ((dyn || WIN) && n_rows == 0 && blockIdx.x == 0 && threadIdx.x == 0 && (forms & EFEM_PATTERN))
            row_ptr_out[0] = 0;
        return;
    }
    constexpr int NS = 1 + 2 * NO, WSEG = 32 * NS, NW = TRI_TPB / 32;
    __shared__ int s_col[NW][WSEG];
    __shared__ double2 s_v[NW][WSEG];  // (M, K) of one entry: one 16-byte store / load
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int* sc = s_col[wid];
    double2* sv = s_v[wid];
    const int nbatch = (n_rows + 31) >> 5;
    const int stride = gridDim.x * NW;
    int batch = blockIdx.x * NW + wid;
    if (batch >= nbatch) return;

    // Pipeline.  Triangles (coordinates held in Ids): four stages -- while
    // batch b is computed, the coordinates of b+1, the element data of b+2 and
    // the records of b+3 are in flight.  Faces (24 doubles of coordinates per
    // pair): three stages -- coordinates of b, element data of b+1, records
    // of b+2.
    constexpr bool DEEP = P::DEEP;
    TriL1 c1 = tri_l1(inc_ptr, rec, batch, nbatch, n_rows, lane);
    TriL1 n1 = tri_l1(inc_ptr, rec, batch + stride, nbatch, n_rows, lane);
    TriL1 n2 = DEEP ? tri_l1(inc_ptr, rec, batch + 2 * stride, nbatch, n_rows, lane) : TriL1{};
    typename P::Ids T0, T1, U0, U1;
    if constexpr (DEEP) {
        P::load_ids(elems, e2d, c1.rr.x, T0);
        P::load_ids2(elems, e2d, c1.rr.y, T1);
        typename P::Geo g;
        P::load_x(coords, gh, T0, g);
        P::load_x2(coords, T1);
        if (batch + stride < nbatch) {
            P::load_ids(elems, e2d, n1.rr.x, U0);
            P::load_ids2(elems, e2d, n1.rr.y, U1);
        }
    } else {
        P::load_ids(elems, e2d, c1.rr.x, T0);
        P::load_ids(elems, e2d, c1.rr.y, T1);
    }

    for (; batch < nbatch; batch += stride) {
        typename P::Geo G0, G1;
        typename P::Ids V0, V1;
        TriL1 n3{};
        const bool has_next = batch + stride < nbatch;
        if constexpr (DEEP) {
            // L3 of b+1, L2 of b+2, L1 of b+3
            if (has_next) {
                P::load_x(coords, gh, U0, G0);
                P::load_x2(coords, U1);
            }
            if (batch + 2 * stride < nbatch) {
                P::load_ids(elems, e2d, n2.rr.x, V0);
                P::load_ids2(elems, e2d, n2.rr.y, V1);
            }
            n3 = tri_l1(inc_ptr, rec, batch + 3 * stride, nbatch, n_rows, lane);
        } else {
            // L3 of b, L2 of b+1, L1 of b+2
            P::load_x(coords, gh, T0, G0);
            P::load_x(coords, gh, T1, G1);
            if (has_next) {
                P::load_ids(elems, e2d, n1.rr.x, U0);
                P::load_ids(elems, e2d, n1.rr.y, U1);
            }
            n3 = tri_l1(inc_ptr, rec, batch + 2 * stride, nbatch, n_rows, lane);
        }

        // ---- batch b
        const int w0 = batch * 32;
        const int li = w0 + lane;
        const bool live = li < n_rows;
        const bool two = c1.rr.x != c1.rr.y;
        const int t = live ? 1 + two : 0;
        // warp prefix of t in {0, 1, 2}: live rows below plus two-element rows
        // below (two ballots and popcounts instead of a shuffle scan)
        const unsigned b_live = __ballot_sync(0xffffffffu, live);
        const unsigned b_two = __ballot_sync(0xffffffffu, live && two);
        const unsigned below = (1u << lane) - 1u;
        const int incl = __popc(b_live & below) + __popc(b_two & below) + t;
        const int ib0 = __shfl_sync(0xffffffffu, c1.ib0, 0);
        const int tot = __popc(b_live) + __popc(b_two);
        const int nr = min(32, n_rows - w0);
        const int gbase = row0 + w0 + NO * ib0 - out_base;
        const int segn = nr + NO * tot;
        const int o = lane + NO * (incl - t);
        if (forms & EFEM_PATTERN) {
            if (live) row_ptr_out[li] = gbase + o;
            if (li == n_rows - 1) row_ptr_out[n_rows] = gbase + segn;
        }
        // (rows of more than two elements are flagged by the symbolic pass)
        const bool bad = false;
        if (!__any_sync(0xffffffffu, bad) && segn <= WSEG) {
            if (live) {
                double m0a, k0a, m0b, k0b, ma[NO], ka[NO], mb[NO], kb[NO];
                int ca[NO], cb[NO];
                if constexpr (DEEP) P::complete2(T0, T1);
                const double da = P::row(T0, G0, gh, c1.rr.x, m0a, k0a, ca, ma, ka);
                const double db = P::row(T1, G1, gh, c1.rr.y, m0b, k0b, cb, mb, kb);
                const bool bad_a = !(fabs(da) > 0.0 && fabs(da) < INFINITY);
                const bool bad_b = two && !(fabs(db) > 0.0 && fabs(db) < INFINITY);
                if (bad_a || bad_b) {
                    atomicOr(&hdr->flags[F_DEGENERATE], 1);
                    atomicMin(&hdr->bad_element, (unsigned long long)((bad_a ? c1.rr.x : c1.rr.y) >> 3));
                }
                int cl[NS];
                double am[NS], ak[NS];
                cl[0] = own_base + li;
                am[0] = two ? m0a + m0b : m0a;
                ak[0] = two ? k0a + k0b : k0a;
#pragma unroll
                for (int q = 0; q < NO; ++q) {
                    cl[1 + q] = ca[q];
                    am[1 + q] = ma[q];
                    ak[1 + q] = ka[q];
                    cl[1 + NO + q] = two ? cb[q] : INT_MAX;
                    am[1 + NO + q] = mb[q];
                    ak[1 + NO + q] = kb[q];
                }
                int rk[NS];
#pragma unroll
                for (int x = 0; x < NS; ++x) rk[x] = 0;
#pragma unroll
                for (int x = 0; x < NS; ++x)
#pragma unroll
                    for (int y = x + 1; y < NS; ++y) {
                        const bool lt = cl[x] < cl[y];
                        rk[y] += lt;
                        rk[x] += !lt;
                    }
#pragma unroll
                for (int x = 0; x < NS; ++x) {
                    if (x <= NO || two) {
                        sc[o + rk[x]] = cl[x];
                        sv[o + rk[x]] = make_double2(am[x], ak[x]);
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < NS; ++u) {
                const int x = u * 32 + lane;
                if (x < segn) {
                    const int gx = gbase + x;
                    const double2 v = sv[x];
                    if (forms & EFEM_PATTERN) col_idx[gx] = sc[x];
                    if (forms & EFEM_MASS) vals_m[gx] = v.x;
                    if (forms & EFEM_STIFF) vals_k[gx] = v.y;
                }
            }
            __syncwarp();
        }
        // rotate the pipeline
        if constexpr (DEEP) {
            c1 = n1;
            n1 = n2;
            n2 = n3;
            T0 = U0;
            T1 = U1;
            U0 = V0;
            U1 = V1;
        } else {
            c1 = n1;
            n1 = n3;
            T0 = U0;
            T1 = U1;
        }
    }
}

// ---------------------------------------------------------------------------------
// 3D edges (NE0).  Row (a, b) with t tets around the edge; tet j = {a, b, c_j,
// d_j}.  Columns are the edges among W = {a, b} U link vertices: ab, a-w and
// b-w for every distinct link vertex w, and c_j-d_j.  Fast path (t <= 7,
// |W| <= 11, node ids < 2^27):
//   W by one 16-key bitonic network in registers (key = node << 5 | source);
//   positions of the sources in a per-thread shared scratch;
//   the row's columns as bits of ONE 64-bit mask over the C(|W|, 2) <= 55
//   lexicographic pairs; a column's slot = popcount of the mask below it;
//   per tet, the slots of its 6 pair types (ab shared) are packed 5 bits each
//   and each local edge picks its slot by the roles of its endpoints.
// Accumulators are column-major in shared memory (slot q of row r at
// q * NUM_TPB + r: bank-conflict free) and flushed in CSR order.  Rows that
// miss the fast-path limits use row_generic (any shape, 256-bit masks).
// ---------------------------------------------------------------------------------
constexpr int NE3_SLOTS = 19;  // staged row length cap (Kuhn max: 19)
constexpr int NE3_LD = NUM_TPB + 1;  // padded column-major stride
constexpr int NE3_TMAX = 7;

__device__ __forceinline__ int pair_index(int p, int q, int nw) {  // p < q
    return p * nw - ((p * (p + 1)) >> 1) + (q - p - 1);
}

// The fast path of one row (see above).  SM: the accumulators are the
// CTA's shared staging columns (stride NE3_LD), so every accumulator access
// is a shared-memory instruction; otherwise they are the row's CSR segment
// in global memory (stride 1, an oversize row in the tile).
// g[i] of a tet's vertex ids held as two 64-bit pairs: one select + one shift
__device__ __forceinline__ int sel4p(unsigned long long g01, unsigned long long g23, int i) {
    const unsigned long long w = (i & 2) ? g23 : g01;
    return (int)(uint32_t)(w >> ((i & 1) * 32));
}

template <class KT, bool SM, int TM>
__device__ __forceinline__ void ne3_fast_row(const double* __restrict__ coords, const int32_t* __restrict__ elems,
                                             const int32_t* __restrict__ inc, const int32_t* __restrict__ e2d,
                                             int own_base, int i, int ib, int t, int rlen, unsigned char* P,
                                             int* ccol, double* cvm, double* cvk, WsHeader* hdr, bool& ok,
                                             bool& done) {
    constexpr int st = SM ? NE3_LD : 1;
    uint32_t key[16];
    int inst[TM], roles[TM], cv[TM], dv[TM];  // cv / dv: each tet's two link vertices (c, d)
    int a = 0, b = 0;
    // all index loads first, then all element loads: two round trips
    // (slots j >= t repeat the last incidence and are masked below)
#pragma unroll
    for (int j = 0; j < TM; ++j) inst[j] = __ldg(inc + ib + min(j, t - 1)) & INST_MASK;
    {   // ascending element id (the symbolic pass groups a node's tets
        // by edge without ordering them): a fixed summation order
        int srt[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) srt[j] = j < t && j < TM ? inst[j] : INT_MAX;
#pragma unroll
        for (int kk = 2; kk <= 8; kk <<= 1)
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1)
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    const int y = x ^ jj;
                    if (y > x) {
                        const int lo = min(srt[x], srt[y]), hi = max(srt[x], srt[y]);
                        const bool asc = (x & kk) == 0;
                        srt[x] = asc ? lo : hi;
                        srt[y] = asc ? hi : lo;
                    }
                }
        // (a select chain, not srt[t - 1]: a dynamic index would put
        // srt in local memory)
        int last = srt[0];
#pragma unroll
        for (int j = 1; j < TM; ++j) last = j == t - 1 ? srt[j] : last;
#pragma unroll
        for (int j = 0; j < TM; ++j) inst[j] = j < t ? srt[j] : last;
    }
    int4 gq[TM];
#pragma unroll
    for (int j = 0; j < TM; ++j) gq[j] = __ldg(reinterpret_cast<const int4*>(elems) + (inst[j] >> 3));
#pragma unroll
    for (int j = 0; j < TM; ++j) {
        const int pe = inst[j];
        const int k = pe & 7;
        const int g[4] = {gq[j].x, gq[j].y, gq[j].z, gq[j].w};
        // local edge k = (s0, s1) (Fig. 1, reading C4) and the other two
        // vertices (lc, ld): 2-bit fields of one byte per k of a 48-bit constant
        const unsigned rk8 = (unsigned)(0x874ec99cd8e4ull >> (8 * k));
        const int s0 = rk8 & 3, s1 = (rk8 >> 2) & 3, lc = (rk8 >> 4) & 3, ld = (rk8 >> 6) & 3;
        const unsigned long long g01 = ((unsigned long long)(uint32_t)g[1] << 32) | (uint32_t)g[0];
        const unsigned long long g23 = ((unsigned long long)(uint32_t)g[3] << 32) | (uint32_t)g[2];
        const int g0 = sel4p(g01, g23, s0), g1 = sel4p(g01, g23, s1);
        const int sw = g0 > g1;  // local vertex s1 carries the row's a
        if (j == 0) {
            a = min(g0, g1);
            b = max(g0, g1);
        }
        // lc, ld (2 bits each) and the local edge ids of the role pairs ac, ad,
        // bc, bd, cd (3 bits each) from a table over (k, swap): Fig. 1 numbering
        const int ti = 2 * k + sw;
        const unsigned long long tw =
            ti < 4 ? 0x542358d0446b4ad1ull : (ti < 8 ? 0x2a21286832253948ull : 0x18981622066a0a99ull);
        const int e5 = (int)((tw >> (16 * (ti & 3))) & 0x7fffull);
        roles[j] = lc | (ld << 2) | (e5 << 4);
        const bool live = j < t;
        cv[j] = sel4p(g01, g23, lc);
        dv[j] = sel4p(g01, g23, ld);
        key[2 * j] = live ? (((uint32_t)cv[j] << 5) | (uint32_t)(2 * j)) : 0xffffffffu;
        key[2 * j + 1] = live ? (((uint32_t)dv[j] << 5) | (uint32_t)(2 * j + 1)) : 0xffffffffu;
    }
#pragma unroll
    for (int x = 2 * TM; x < 14; ++x) key[x] = 0xffffffffu;  // (unused slots when TM < 7)
    key[14] = ((uint32_t)a << 5) | 14u;
    key[15] = ((uint32_t)b << 5) | 15u;
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
    int rk = -1;
    uint32_t prev = 0xffffffffu;
#pragma unroll
    for (int x = 0; x < 16; ++x) {
        if (key[x] != 0xffffffffu) {
            const uint32_t v = key[x] >> 5;
            rk += v != prev;
            prev = v;
            P[(key[x] & 31u) * NUM_TPB] = (unsigned char)rk;
        }
    }
    const int nw = rk + 1;
    if (nw <= 11) {
        const int pa = P[14 * NUM_TPB], pb = P[15 * NUM_TPB];
        const int iab = pair_index(pa, pb, nw);
        // column mask over lexicographic pairs of W positions
        unsigned long long mask = 1ull << iab;
        int pidx[TM];  // packed pair indices: ac | ad << 6 | bc << 12 | bd << 18 | cd << 24
#pragma unroll
        for (int j = 0; j < TM; ++j) {
            if (j < t) {
                const int pc = P[(2 * j) * NUM_TPB], pd = P[(2 * j + 1) * NUM_TPB];
                const int iac = pair_index(min(pa, pc), max(pa, pc), nw);
                const int iad = pair_index(min(pa, pd), max(pa, pd), nw);
                const int ibc = pair_index(min(pb, pc), max(pb, pc), nw);
                const int ibd = pair_index(min(pb, pd), max(pb, pd), nw);
                const int icd = pair_index(min(pc, pd), max(pc, pd), nw);
                mask |= (1ull << iac) | (1ull << iad) | (1ull << ibc) | (1ull << ibd) | (1ull << icd);
                pidx[j] = iac | (iad << 6) | (ibc << 12) | (ibd << 18) | (icd << 24);
            }
        }
        ok = __popcll(mask) == rlen;
        done = true;
        if (ok) {
            // Accumulation with fewer shared-memory accesses (their slots are
            // data dependent, so most of them meet bank conflicts): the own
            // column ab, held by every tet, sums in registers; every other
            // column is stored by its first tet (0.0 + v, what a zeroed
            // accumulator would hold) and read-modify-written by the later
            // ones -- the same sums in the same order, bit for bit.
            const int sab = __popcll(mask & ((1ull << iab) - 1ull));
            unsigned long long seen = 1ull << iab;
            double dm = 0.0, dk = 0.0;
            // role frame: vertices ordered (a, b, c, d), a < b the row's
            // edge.  The globally oriented Whitney basis of edge {x, y}
            // is sigma_xy (l_x grad l_y - l_y grad l_x), sigma_xy = +1
            // iff x < y, which is exactly s_k times the paper's mapped
            // local basis, so no other signs enter.
            // With n_v the area normals (adjugate rows) and N_uv = n_u.n_v,
            // G = N / det^2:
            //   M_(ab)(pq) = |K|/20 [(1+d_ap)G_bq - (1+d_aq)G_bp - (1+d_bp)G_aq + (1+d_bq)G_ap]
            //   K_(ab)(pq) = 4 |K| (G_ap G_bq - G_aq G_bp)
            double xa[3], xb[3];
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                xa[cc] = __ldg(coords + a * 3 + cc);
                xb[cc] = __ldg(coords + b * 3 + cc);
            }
#pragma unroll
            for (int j = 0; j < TM; ++j) {
                if (j < t) {
                    const int e = inst[j] >> 3;
                    const int rl = roles[j];
                    const int e5 = rl >> 4;
                    const int c = cv[j], d = dv[j];  // (kept from the first pass: no second tet load)
                    double e1[3], e2[3], e3[3];
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) {
                        e1[cc] = xb[cc] - xa[cc];
                        e2[cc] = __ldg(coords + c * 3 + cc) - xa[cc];
                        e3[cc] = __ldg(coords + d * 3 + cc) - xa[cc];
                    }
                    const double nb[3] = {e2[1] * e3[2] - e2[2] * e3[1], e2[2] * e3[0] - e2[0] * e3[2],
                                          e2[0] * e3[1] - e2[1] * e3[0]};
                    const double nc[3] = {e3[1] * e1[2] - e3[2] * e1[1], e3[2] * e1[0] - e3[0] * e1[2],
                                          e3[0] * e1[1] - e3[1] * e1[0]};
                    const double nd[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                                          e1[0] * e2[1] - e1[1] * e2[0]};
                    const double det = e1[0] * nb[0] + e1[1] * nb[1] + e1[2] * nb[2];
                    if (!(det != 0.0) || !isfinite(det)) {
                        atomicOr(&hdr->flags[F_DEGENERATE], 1);
                        atomicMin(&hdr->bad_element, (unsigned long long)e);
                    }
                    const double na[3] = {-(nb[0] + nc[0] + nd[0]), -(nb[1] + nc[1] + nd[1]),
                                          -(nb[2] + nc[2] + nd[2])};
                    auto dot = [](const double* u, const double* v) { return u[0] * v[0] + u[1] * v[1] + u[2] * v[2]; };
                    const double Naa = dot(na, na), Nbb = dot(nb, nb), Nab = dot(na, nb);
                    const double Nac = dot(na, nc), Nad = dot(na, nd), Nbc = dot(nb, nc), Nbd = dot(nb, nd);
                    const double rd = 1.0 / fabs(det);
                    const double cm = rd * (1.0 / 120.0);
                    const double ck = (2.0 / 3.0) * rd * rd * rd;
                    // role columns ab ac ad bc bd cd
                    const int pc = P[(2 * j) * NUM_TPB], pd = P[(2 * j + 1) * NUM_TPB];
                    // orientation signs as sign-bit flips ((+-cm) x == +-(cm x) exactly)
                    auto sgn = [](bool pos, double v) {
                        return __longlong_as_double(__double_as_longlong(v) ^ ((unsigned long long)!pos << 63));
                    };
                    const bool sac = pa < pc, sad = pa < pd, sbc = pb < pc, sbd = pb < pd, scd = pc < pd;
                    const double vm[6] = {cm * (2.0 * (Naa + Nbb - Nab)),
                                          sgn(sac, cm * (2.0 * Nbc - Nab - Nac + Naa)),
                                          sgn(sad, cm * (2.0 * Nbd - Nab - Nad + Naa)),
                                          sgn(sbc, cm * (Nbc - Nbb - 2.0 * Nac + Nab)),
                                          sgn(sbd, cm * (Nbd - Nbb - 2.0 * Nad + Nab)),
                                          sgn(scd, cm * (Nbd - Nbc - Nad + Nac))};
                    const double vk[6] = {ck * (Naa * Nbb - Nab * Nab),
                                          sgn(sac, ck * (Naa * Nbc - Nac * Nab)),
                                          sgn(sad, ck * (Naa * Nbd - Nad * Nab)),
                                          sgn(sbc, ck * (Nab * Nbc - Nac * Nbb)),
                                          sgn(sbd, ck * (Nab * Nbd - Nad * Nbb)),
                                          sgn(scd, ck * (Nac * Nbd - Nad * Nbc))};
                    // DOF ids of the role pairs ac ad bc bd cd (local edge ids packed with
                    // the roles in the first pass)
                    const int32_t* de = e2d + e * 6;
                    const int pi = pidx[j];
                    dm += vm[0];
                    dk += vk[0];
#pragma unroll
                    for (int u = 1; u < 6; ++u) {
                        // rank of the column's bit among the row's: popcount of the
                        // bits below it (mask shifted up: no 64-bit subtract / and)
                        const int pb_ = (pi >> (6 * (u - 1))) & 63;
                        const int slot = (pb_ ? __popcll(mask << (64 - pb_)) : 0) * st;
                        const unsigned long long bit = 1ull << pb_;
                        const bool first = !(seen & bit);
                        seen |= bit;
                        if (first) ccol[slot] = __ldg(de + ((e5 >> (3 * (u - 1))) & 7));
                        const double om = first ? 0.0 : cvm[slot];
                        const double ok_ = first ? 0.0 : cvk[slot];
                        cvm[slot] = om + vm[u];
                        cvk[slot] = ok_ + vk[u];
                    }
                }
            }
            ccol[sab * st] = own_base + i;
            cvm[sab * st] = dm;
            cvk[sab * st] = dk;
        }
    }
}

template <class KT>
__global__ void __launch_bounds__(NUM_TPB, 512 / NUM_TPB) k_rows_ne3(const double* __restrict__ coords,
                                                      const int32_t* __restrict__ elems,
                                                      const int32_t* __restrict__ inc_ptr,
                                                      const int32_t* __restrict__ inc,
                                                      const int32_t* __restrict__ e2d,
                                                      const int32_t* __restrict__ row_ptr, int n_rows_arg,
                                                      int own_base, int out_base,
                                                      unsigned forms, int fast_ids, int32_t* __restrict__ row_ptr_out,
                                                      int32_t* __restrict__ col_idx,
                                                      double* __restrict__ vals_m, double* __restrict__ vals_k,
                                                      WsHeader* hdr, int dyn, long long cap_nnz,
                                                      const long long* __restrict__ win) {
    static_assert(KT::D == 3 && !KT::FACES, "NE0 3D only");
    // node ids out of range (flagged by the enumeration): nothing is gathered
    if (*(volatile const int*)&hdr->flags[F_INVALID_NODE]) return;
    int n_rows = dyn ? dyn_rows(hdr, n_rows_arg, cap_nnz) : n_rows_arg;
    if (win) {
        n_rows = win_rows(hdr, win, n_rows_arg, cap_nnz);
        if (n_rows > 0) {
            const int r0 = (int)win[0];
            out_base = (int)win[2];
            own_base = (int)win[4];
            inc_ptr += r0;
            row_ptr += r0;
        }
    }
    if (n_rows <= 0 || (int)(blockIdx.x * NUM_TPB) >= n_rows) {
        if ((dyn || win) && n_rows == 0 && blockIdx.x == 0 && threadIdx.x == 0 && (forms & EFEM_PATTERN))
            row_ptr_out[0] = 0;
        return;
    }
    extern __shared__ __align__(16) unsigned char ne3_smem[];
    double* s_vm = reinterpret_cast<double*>(ne3_smem);
    double* s_vk = s_vm + NE3_SLOTS * NE3_LD;
    int* s_col = reinterpret_cast<int*>(s_vk + NE3_SLOTS * NE3_LD);
    int* s_off = s_col + NE3_SLOTS * NE3_LD;  // NUM_TPB + 1 row offsets
    unsigned short* s_map = reinterpret_cast<unsigned short*>(s_off + NUM_TPB + 1);  // CSR position -> slot
    unsigned char* s_pos = reinterpret_cast<unsigned char*>(s_map + NE3_SLOTS * NUM_TPB);  // 16 per thread

#if EFEM_NE3_WARPFLUSH
    // every warp stages and flushes its own 32 rows (their CSR segment is
    // contiguous): no CTA barrier between warps of unequal work
    const int wq = (int)(threadIdx.x >> 5);
    const int r0 = blockIdx.x * NUM_TPB + 32 * wq;
    if (r0 >= n_rows) return;
    const int nr = min(32, n_rows - r0);
    unsigned short* const wmap = s_map + wq * (NE3_SLOTS * 32);
    constexpr int FL_N = 32;
    const int fl_i = (int)(threadIdx.x & 31);
#else
    const int r0 = blockIdx.x * NUM_TPB;
    const int nr = min(NUM_TPB, n_rows - r0);
    unsigned short* const wmap = s_map;
    constexpr int FL_N = NUM_TPB;
    const int fl_i = (int)threadIdx.x;
#endif
    const int seg0 = __ldg(row_ptr + r0);
    const int segn = __ldg(row_ptr + r0 + nr) - seg0;
    const int i = r0 + fl_i;
    int rlen = 0, ib = 0, t = 0;
    if (i < n_rows) {
        const int rb = __ldg(row_ptr + i);
        rlen = __ldg(row_ptr + i + 1) - rb;
        if (forms & EFEM_PATTERN) {
            row_ptr_out[i] = rb - out_base;
            if (i == n_rows - 1) row_ptr_out[n_rows] = rb + rlen - out_base;
        }
        s_off[threadIdx.x] = rb - seg0;
        ib = __ldg(inc_ptr + i);
        t = __ldg(inc_ptr + i + 1) - ib;
    }
#if EFEM_NE3_WARPFLUSH
    const bool staged = __all_sync(0xffffffffu, rlen <= NE3_SLOTS);
#else
    const bool staged = __syncthreads_and(rlen <= NE3_SLOTS);
#endif

    if (i < n_rows) {
        int* ccol;
        double *cvm, *cvk;
        int st;
        if (staged) {
            ccol = s_col + threadIdx.x;
            cvm = s_vm + threadIdx.x;
            cvk = s_vk + threadIdx.x;
            st = NE3_LD;
        } else {  // an oversize row in the tile: accumulate in place in global memory
            const int rb = s_off[threadIdx.x] + seg0 - out_base;
            ccol = col_idx + rb;
            cvm = vals_m ? vals_m + rb : s_vm + threadIdx.x;
            cvk = vals_k ? vals_k + rb : s_vk + threadIdx.x;
            st = 1;
        }
        bool ok = false, done = false;
        if (fast_ids && t >= 1 && t <= NE3_TMAX) {
            unsigned char* P = s_pos + threadIdx.x;  // P[src * NUM_TPB]
            // (rows of <= 6 tets -- every row of a structured tet mesh -- take a
            // 6-slot instantiation: fewer live registers)
            if (staged && t <= 6)
                ne3_fast_row<KT, true, 6>(coords, elems, inc, e2d, own_base, i, ib, t, rlen, P, s_col + threadIdx.x,
                                          s_vm + threadIdx.x, s_vk + threadIdx.x, hdr, ok, done);
            else if (staged)
                ne3_fast_row<KT, true, NE3_TMAX>(coords, elems, inc, e2d, own_base, i, ib, t, rlen, P,
                                                 s_col + threadIdx.x, s_vm + threadIdx.x, s_vk + threadIdx.x, hdr, ok,
                                                 done);
            else
                ne3_fast_row<KT, false, NE3_TMAX>(coords, elems, inc, e2d, own_base, i, ib, t, rlen, P, ccol, cvm,
                                                  cvk, hdr, ok, done);
        }
        if (!done) ok = row_generic<KT>(coords, elems, inc, e2d, ib, t, rlen, ccol, cvm, cvk, st, hdr);
        if (!ok) atomicOr(&hdr->flags[F_ROW_MISMATCH], 1);
        if (staged) {
            const int off = s_off[threadIdx.x];
#pragma unroll
            for (int q = 0; q < NE3_SLOTS; ++q)
                if (q < rlen) wmap[off + q] = (unsigned short)(q * NE3_LD + threadIdx.x);
        }
    }
    if (!staged) return;
#if EFEM_NE3_WARPFLUSH
    __syncwarp();
#else
    __syncthreads();
#endif
    // coalesced flush in CSR order through the position -> slot map
    for (int x = fl_i; x < segn; x += FL_N) {
        const int src = wmap[x];
        const int gx = seg0 - out_base + x;
        if (forms & EFEM_PATTERN) col_idx[gx] = s_col[src];
        if (forms & EFEM_MASS) vals_m[gx] = s_vm[src];
        if (forms & EFEM_STIFF) vals_k[gx] = s_vk[src];
    }
}

constexpr size_t NE3_SMEM = (size_t)NE3_SLOTS * NE3_LD * (8 + 8 + 4) + (NUM_TPB + 1) * 4 +
                            (size_t)NE3_SLOTS * NUM_TPB * 2 + 16 * NUM_TPB;

// ---------------------------------------------------------------------------------
template <class KT>
efem_status launch_rows(Plan& p, unsigned forms, efem_csr* out, const RowWindow& w, cudaStream_t s) {
    if (w.n_rows == 0) return EFEM_OK;
    double* vm = (forms & EFEM_MASS) ? out->vals_mass : nullptr;
    double* vk = (forms & EFEM_STIFF) ? out->vals_stiff : nullptr;
    // (a device window offsets the arrays inside the kernel)
    const int32_t* inc_ptr = p.inc_ptr + (w.win ? 0 : w.row0);
    const int32_t* row_ptr = p.row_ptr + (w.win ? 0 : w.row0);
    if constexpr (KT::D == 2 || KT::FACES) {
        using P = std::conditional_t<KT::D == 2, TriPolicy, FacePolicy>;
#ifndef EFEM_TRI_MINB
#define EFEM_TRI_MINB 2
#endif
        constexpr int MINB = EFEM_TRI_MINB;
        auto launch = [&](auto kern) -> efem_status {
            // persistent grid = SMs x resident CTAs, per device (cached)
            static std::atomic<int> grids[kMaxDevices];
            int dev = 0;
            EFEM_CUDA_TRY(cudaGetDevice(&dev));
            int grid = dev < kMaxDevices ? grids[dev].load(std::memory_order_relaxed) : 0;
            if (!grid) {
                int sms = 0, per_sm = 0;
                EFEM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
                EFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TRI_TPB, 0));
                grid = sms * (per_sm > 0 ? per_sm : 1);
                if (dev < kMaxDevices) grids[dev].store(grid, std::memory_order_relaxed);
            }
            const int64_t need = (w.n_rows + TRI_TPB - 1) / TRI_TPB;
            kern<<<(unsigned)(need < grid ? need : grid), TRI_TPB, 0, s>>>(
                p.coords, p.elems, inc_ptr, p.rec + (w.win ? 0 : w.row0), w.e2d, (int)w.row0, (int)w.n_rows,
                w.own_base, w.out_base, forms, out->row_ptr, out->col_idx, vm, vk, p.hdr, (int)w.dyn,
                (long long)w.cap_nnz, w.win, w.gh);
            return EFEM_OK;
        };
        efem_status st;
        if constexpr (KT::D == 2) {
            if (w.ghost) {
                st = w.win ? launch(k_rows_tri<KT, GhostDeepPolicy, MINB, true>)
                           : launch(k_rows_tri<KT, GhostDeepPolicy, MINB, false>);
                if (st != EFEM_OK) return st;
                EFEM_LAUNCH_CHECK();
                return EFEM_OK;
            }
        }
        st = w.win ? launch(k_rows_tri<KT, P, MINB, true>) : launch(k_rows_tri<KT, P, MINB, false>);
        if (st != EFEM_OK) return st;
    } else {
        const int fast_ids = p.n_nodes < (1ll << 27);
        static std::atomic<bool> attr[kMaxDevices];  // the smem opt-in is per device
        int dev = 0;
        EFEM_CUDA_TRY(cudaGetDevice(&dev));
        if (dev >= kMaxDevices || !attr[dev].load(std::memory_order_relaxed)) {
            EFEM_CUDA_TRY(cudaFuncSetAttribute(k_rows_ne3<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)NE3_SMEM));
            if (dev < kMaxDevices) attr[dev].store(true, std::memory_order_relaxed);
        }
        k_rows_ne3<KT><<<grid_for(w.n_rows, NUM_TPB), NUM_TPB, NE3_SMEM, s>>>(p.coords, p.elems, inc_ptr, p.bucket, w.e2d, row_ptr,
                                                       (int)w.n_rows, w.own_base, w.out_base, forms, fast_ids,
                                                       out->row_ptr, out->col_idx, vm, vk, p.hdr, (int)w.dyn,
                                                       (long long)w.cap_nnz, w.win);
    }
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status launch_rows_any(Plan& p, unsigned forms, efem_csr* out, const RowWindow& w, cudaStream_t s) {
    if (p.dim == 2) return p.element == EFEM_RT0 ? launch_rows<Kind<2, EFEM_RT0>>(p, forms, out, w, s)
                                                 : launch_rows<Kind<2, EFEM_NED0>>(p, forms, out, w, s);
    return p.element == EFEM_RT0 ? launch_rows<Kind<3, EFEM_RT0>>(p, forms, out, w, s)
                                 : launch_rows<Kind<3, EFEM_NED0>>(p, forms, out, w, s);
}

}  // namespace efem
