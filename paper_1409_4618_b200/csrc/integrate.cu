// integrate.cu -- SURVEY.md §8(f) rows f1 / f2 on the GPU: the paper's
// vectorized integration (Sec. 3.1) -- degree-6
// quadrature points F_K(xh_i) of all elements, load vectors against the
// global Piola-mapped basis, L2 norms and field errors -- plus the CSR SpMV
// and the Jacobi-preconditioned CG used by the eddy-current example
// (PAPER.md:863-918).  Every reduction runs in a fixed order (per-element
// values, then a two-level tree), so results are bitwise reproducible.
// Product path only; shares nothing with oracle/.
#include <atomic>
#include <cmath>
#include <vector>

#include "element.cuh"

namespace efem {

// ---- degree-6 rules: Dunavant 12-point (2D), Keast
// 24-point (3D); barycentric (l1, l2[, l3]) and weights including |K_hat|.
struct Quad6 {
    double l[24][3];
    double w[24];
    int nq;
};

__constant__ Quad6 c_quad[2];  // [0] 2D, [1] 3D

namespace {

Quad6 make_quad6(int dim) {
    Quad6 Q{};
    int n = 0;
    auto put = [&](double a, double b, double c, double wt) {
        Q.l[n][0] = a;
        Q.l[n][1] = b;
        Q.l[n][2] = c;
        Q.w[n] = wt;
        ++n;
    };
    if (dim == 2) {
        struct S3 { double w, a, b; };
        const S3 s3[2] = {{0.116786275726379, 0.501426509658179, 0.249286745170910},
                          {0.050844906370207, 0.873821971016996, 0.063089014491502}};
        for (const S3& s : s3) {  // (l0, l1, l2) in {(a,b,b), (b,a,b), (b,b,a)}
            put(s.b, s.b, 0.0, 0.5 * s.w);
            put(s.a, s.b, 0.0, 0.5 * s.w);
            put(s.b, s.a, 0.0, 0.5 * s.w);
        }
        // the six placements of (c0, c1, c2) on (l0, l1, l2), permutations in
        // lexicographic order (the point order is part of the interface: fq
        // rows follow it)
        const double v[3] = {0.053145049844817, 0.310352451033784, 0.636502499121399};
        const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        for (int i = 0; i < 6; ++i) put(v[perm[i][1]], v[perm[i][2]], 0.0, 0.5 * 0.082851075618374);
    } else {
        const double a4[3] = {0.214602871259151684, 0.0406739585346113397, 0.322337890142275646};
        const double w4[3] = {0.0399227502581679, 0.0100772110553207, 0.0553571815436544};
        for (int c = 0; c < 3; ++c) {
            const double a = a4[c], b = 1.0 - 3.0 * a, wt = w4[c] / 6.0;
            put(a, a, a, wt);
            put(b, a, a, wt);
            put(a, b, a, wt);
            put(a, a, b, wt);
        }
        const double a = 0.0636610018750175299, b = 0.269672331458315867, c = 0.603005664791649076;
        const double wt = 0.0482142857142857 / 6.0;
        // the 12 arrangements of {a, a, b, c} on (l0..l3): a at slots i0 < i1,
        // b at i2, c at i3, (i0, i1, i2, i3) in lexicographic order
        for (int i0 = 0; i0 < 4; ++i0)
            for (int i1 = i0 + 1; i1 < 4; ++i1)
                for (int i2 = 0; i2 < 4; ++i2) {
                    if (i2 == i0 || i2 == i1) continue;
                    const int i3 = 6 - i0 - i1 - i2;
                    double lam[4];
                    lam[i0] = a;
                    lam[i1] = a;
                    lam[i2] = b;
                    lam[i3] = c;
                    put(lam[1], lam[2], lam[3], wt);
                }
    }
    Q.nq = n;
    return Q;
}

std::atomic<bool> g_quad_ready[64];

// __constant__ memory is per device: the tables are uploaded once per device
efem_status ensure_quad() {
    int dev = 0;
    EFEM_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 64 && g_quad_ready[dev].load(std::memory_order_acquire)) return EFEM_OK;
    Quad6 q[2] = {make_quad6(2), make_quad6(3)};
    EFEM_CUDA_TRY(cudaMemcpyToSymbol(c_quad, q, sizeof(q)));
    if (dev < 64) g_quad_ready[dev].store(true, std::memory_order_release);
    return EFEM_OK;
}

// ---- element geometry: B = [x1-x0 | x2-x0 (| x3-x0)]
template <int D>
struct Geo {
    double x0[D];
    double B[D][D];  // B[r][c]
    double det;
    double BiT[D][D];  // B^{-T}
};

template <int D>
__device__ __forceinline__ void load_geo(const double* __restrict__ coords, const int (&g)[D + 1], Geo<D>& G) {
    double X[D + 1][D];
#pragma unroll
    for (int v = 0; v <= D; ++v)
#pragma unroll
        for (int c = 0; c < D; ++c) X[v][c] = __ldg(coords + (int64_t)g[v] * D + c);
#pragma unroll
    for (int r = 0; r < D; ++r) {
        G.x0[r] = X[0][r];
#pragma unroll
        for (int c = 0; c < D; ++c) G.B[r][c] = X[c + 1][r] - X[0][r];
    }
    if constexpr (D == 2) {
        G.det = G.B[0][0] * G.B[1][1] - G.B[0][1] * G.B[1][0];
        const double id = 1.0 / G.det;
        G.BiT[0][0] = G.B[1][1] * id;
        G.BiT[0][1] = -G.B[1][0] * id;
        G.BiT[1][0] = -G.B[0][1] * id;
        G.BiT[1][1] = G.B[0][0] * id;
    } else {
        double cof[3][3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int r1 = (r + 1) % 3, r2 = (r + 2) % 3, c1 = (c + 1) % 3, c2 = (c + 2) % 3;
                cof[r][c] = G.B[r1][c1] * G.B[r2][c2] - G.B[r1][c2] * G.B[r2][c1];
            }
        G.det = G.B[0][0] * cof[0][0] + G.B[0][1] * cof[0][1] + G.B[0][2] * cof[0][2];
        const double id = 1.0 / G.det;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) G.BiT[r][c] = cof[r][c] * id;
    }
}

// Reference basis value of local DOF k at xh (PAPER.md:228-238 RT with the
// 3D RT basis doubled (reading C1), 275-289 Ned) and its reference div /
// curl (constant).
template <class KT>
__device__ __forceinline__ void ref_value(int k, const double* xh, double (&v)[KT::D]) {
    const double x1 = xh[0], x2 = xh[1];
    if constexpr (KT::D == 2 && KT::ELEMENT == EFEM_RT0) {
        v[0] = k == 1 ? x1 - 1.0 : x1;
        v[1] = k == 2 ? x2 - 1.0 : x2;
    } else if constexpr (KT::D == 2) {
        v[0] = k == 2 ? 1.0 - x2 : -x2;
        v[1] = k == 1 ? x1 - 1.0 : x1;
    } else if constexpr (KT::FACES) {
        const double x3 = xh[2];
        v[0] = 2.0 * (k == 2 ? x1 - 1.0 : x1);
        v[1] = 2.0 * (k == 1 ? x2 - 1.0 : x2);
        v[2] = 2.0 * (k == 0 ? x3 - 1.0 : x3);
    } else {
        const double x3 = xh[2];
        switch (k) {
            case 0: v[0] = 1.0 - x3 - x2; v[1] = x1; v[2] = x1; break;
            case 1: v[0] = x2; v[1] = 1.0 - x3 - x1; v[2] = x2; break;
            case 2: v[0] = x3; v[1] = x3; v[2] = 1.0 - x2 - x1; break;
            case 3: v[0] = -x2; v[1] = x1; v[2] = 0.0; break;
            case 4: v[0] = 0.0; v[1] = -x3; v[2] = x2; break;
            default: v[0] = x3; v[1] = 0.0; v[2] = -x1; break;
        }
    }
}

template <class KT>
__host__ __device__ constexpr int n_deriv() { return (KT::D == 3 && KT::ELEMENT == EFEM_NED0) ? 3 : 1; }

template <class KT>
__device__ __forceinline__ void ref_deriv(int k, double (&d)[n_deriv<KT>()]) {
    if constexpr (KT::D == 2) {
        d[0] = 2.0;  // div (RT) and curl (Ned) of every 2D reference function
    } else if constexpr (KT::FACES) {
        d[0] = 6.0;
    } else {  // curl of the 3D Ned reference functions
        const double c[6][3] = {{0, -2, 2}, {2, 0, -2}, {-2, 2, 0}, {0, 0, 2}, {2, 0, 0}, {0, 2, 0}};
#pragma unroll
        for (int r = 0; r < 3; ++r) d[r] = c[0][r];
#pragma unroll
        for (int j = 1; j < 6; ++j)
            if (k == j) {
#pragma unroll
                for (int r = 0; r < 3; ++r) d[r] = c[j][r];
            }
    }
}

// Global basis of local DOF k on the element (PAPER.md:240-245, 291-301,
// 323-331): RT s/det B eta, div s/det div; Ned s B^{-T} eta, curl s/det curl
// (2D), s/det B curl (3D).
template <class KT>
__device__ __forceinline__ void global_value(const Geo<KT::D>& G, double s, int k, const double* xh,
                                             double (&phi)[KT::D]) {
    constexpr int D = KT::D;
    double v[D];
    ref_value<KT>(k, xh, v);
#pragma unroll
    for (int r = 0; r < D; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) acc += (KT::ELEMENT == EFEM_RT0 ? G.B[r][c] : G.BiT[r][c]) * v[c];
        phi[r] = KT::ELEMENT == EFEM_RT0 ? s * acc / G.det : s * acc;
    }
}

template <class KT>
__device__ __forceinline__ void global_deriv(const Geo<KT::D>& G, double s, int k, double (&dphi)[n_deriv<KT>()]) {
    double d[n_deriv<KT>()];
    ref_deriv<KT>(k, d);
    if constexpr (n_deriv<KT>() == 3) {
#pragma unroll
        for (int r = 0; r < 3; ++r) dphi[r] = s * (G.B[r][0] * d[0] + G.B[r][1] * d[1] + G.B[r][2] * d[2]) / G.det;
    } else {
        dphi[0] = s * d[0] / G.det;
    }
}

__device__ __forceinline__ const Quad6& quad(int D) { return c_quad[D - 2]; }

// ---- kernels ------------------------------------------------------------------------
// One thread per element (its vertices gathered once), the CTA's points staged
// in shared memory and stored coalesced.
constexpr int QP_TPB = 128;
template <int D>
__global__ void __launch_bounds__(QP_TPB) k_quad_points(const double* __restrict__ coords,
                                                        const int32_t* __restrict__ elems, int64_t n_elems,
                                                        double* __restrict__ pts) {
    const Quad6& Q = quad(D);
    constexpr int NQ = D == 2 ? 12 : 24;
    constexpr int PER = NQ * D;  // doubles per element
    constexpr int LD = PER + 1;  // padded row (odd stride: no shared-memory bank conflicts)
    extern __shared__ double s_pts[];  // QP_TPB * LD
    const int64_t e0 = (int64_t)blockIdx.x * QP_TPB;
    const int64_t e = e0 + threadIdx.x;
    if (e < n_elems) {
        double X[D + 1][D];
#pragma unroll
        for (int v = 0; v <= D; ++v) {
            const int gv = __ldg(elems + e * (D + 1) + v);
#pragma unroll
            for (int c = 0; c < D; ++c) X[v][c] = __ldg(coords + (int64_t)gv * D + c);
        }
#pragma unroll 4
        for (int q = 0; q < NQ; ++q) {
#pragma unroll
            for (int c = 0; c < D; ++c) {
                double x = X[0][c];
#pragma unroll
                for (int v = 1; v <= D; ++v) x += (X[v][c] - X[0][c]) * Q.l[q][v - 1];
                s_pts[threadIdx.x * LD + q * D + c] = x;
            }
        }
    }
    __syncthreads();
    const int64_t cnt = (n_elems - e0 < QP_TPB ? n_elems - e0 : QP_TPB) * PER;
    for (int x = threadIdx.x; x < cnt; x += QP_TPB) pts[e0 * PER + x] = s_pts[(x / PER) * LD + x % PER];
}


// A CTA's per-element input rows (per doubles each, contiguous in src) into
// shared memory rows of odd stride ld: coalesced loads, conflict-free
// per-thread reads afterwards.  (row, col) advance incrementally: no division
// in the loop.
__device__ __forceinline__ void stage_rows(const double* __restrict__ src, int64_t cnt, int per, int ld,
                                           double* __restrict__ dst) {
    const int step_r = blockDim.x / per, step_c = blockDim.x % per;
    int r = threadIdx.x / per, c = threadIdx.x % per;
    constexpr int U = 8;  // loads in flight per thread
    for (int64_t x0 = threadIdx.x; x0 < cnt; x0 += (int64_t)U * blockDim.x) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t x = x0 + (int64_t)u * blockDim.x;
            v[u] = x < cnt ? __ldg(src + x) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (x0 + (int64_t)u * blockDim.x < cnt) dst[r * ld + c] = v[u];
            r += step_r;
            c += step_c;
            if (c >= per) {
                c -= per;
                ++r;
            }
        }
    }
}

// Load vector, element-parallel half: every element's m local contributions
// l_k = sum_q w_q |det| f(x_q) . phi_k(x_q) (the same arithmetic, in the same
// order, as the row-owner loop it replaces), its point values staged.
template <class KT, int PAIR, int TPB>
__global__ void __launch_bounds__(TPB) k_load_elem(const double* __restrict__ coords,
                                                   const int32_t* __restrict__ elems, int64_t n_elems,
                                                   const double* __restrict__ fq, double* __restrict__ loc) {
    constexpr int D = KT::D, NV = KT::NV, M = KT::M;
    constexpr int ND = n_deriv<KT>();
    constexpr int NF = PAIR == 0 ? D : ND;
    constexpr int NQ = D == 2 ? 12 : 24;
    constexpr int PER = NQ * NF, LD = PER | 1;
    extern __shared__ double s_f[];  // TPB * LD
    const Quad6& Q = quad(D);
    const int64_t e0 = (int64_t)blockIdx.x * TPB;
    const int64_t ne = n_elems - e0 < TPB ? n_elems - e0 : TPB;
    const int64_t e = e0 + threadIdx.x;
    int g[NV];
    Geo<D> G;
    if (e < n_elems) {
        load_g<KT>(elems, (int)e, g);
        load_geo<D>(coords, g, G);
    }
    stage_rows(fq + e0 * PER, ne * PER, PER, LD, s_f);
    __syncthreads();
    if (e >= n_elems) return;
    const double adet = fabs(G.det);
    const double* f = s_f + threadIdx.x * LD;
#pragma unroll
    for (int k = 0; k < M; ++k) {
        const double sk = sign_d<KT>(g, k);
        double l = 0.0;
        if constexpr (PAIR == 1) {
            double dphi[ND];
            global_deriv<KT>(G, sk, k, dphi);
#pragma unroll 4
            for (int q = 0; q < NQ; ++q) {
                double dot = 0.0;
#pragma unroll
                for (int c = 0; c < NF; ++c) dot += f[q * NF + c] * dphi[c];
                l += Q.w[q] * adet * dot;
            }
        } else {
#pragma unroll 4
            for (int q = 0; q < NQ; ++q) {
                double phi[D];
                global_value<KT>(G, sk, k, Q.l[q], phi);
                double dot = 0.0;
#pragma unroll
                for (int c = 0; c < NF; ++c) dot += f[q * NF + c] * phi[c];
                l += Q.w[q] * adet * dot;
            }
        }
        loc[e * M + k] = l;
    }
}

// Load vector, row-owner half: b_i = sum of the local contributions of the
// DOF's elements in ascending element order (registers for t <= 4).
template <class KT>
__global__ void __launch_bounds__(256) k_load_gather(const int32_t* __restrict__ inc_ptr,
                                                     const int32_t* __restrict__ inc, int64_t n_dofs,
                                                     const double* __restrict__ loc, double* __restrict__ b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_dofs) return;
    const int ib = __ldg(inc_ptr + i), t = __ldg(inc_ptr + i + 1) - ib;
    double acc = 0.0;
    if (t <= 4) {
        int w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = j < t ? (__ldg(inc + ib + j) & INST_MASK) : INT_MAX;
#pragma unroll
        for (int x = 0; x < 4; ++x)  // (a 4-element sorting network: 6 exchanges)
#pragma unroll
            for (int y = x + 1; y < 4; ++y) {
                const int lo = min(w[x], w[y]), hi = max(w[x], w[y]);
                w[x] = lo;
                w[y] = hi;
            }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < t) acc += __ldg(loc + (int64_t)(w[j] >> 3) * KT::M + (w[j] & 7));
    } else {
        int prev = -1;  // ascending element order by repeated minimum search (t is small)
        for (int j = 0; j < t; ++j) {
            int best = INT_MAX;
            for (int u = 0; u < t; ++u) {
                const int v = __ldg(inc + ib + u) & INST_MASK;
                if (v > prev && v < best) best = v;
            }
            acc += __ldg(loc + (int64_t)(best >> 3) * KT::M + (best & 7));
            prev = best;
        }
    }
    b[i] = acc;
}

constexpr int NORM_TPB = 128;
template <int D>
__global__ void __launch_bounds__(NORM_TPB) k_norm_elem_staged(const double* __restrict__ coords,
                                                               const int32_t* __restrict__ elems, int64_t n_elems,
                                                               const double* __restrict__ fq, int nf,
                                                               double* __restrict__ per_elem) {
    const Quad6& Q = quad(D);
    constexpr int NQ = D == 2 ? 12 : 24;
    const int per = NQ * nf, ld = per | 1;
    extern __shared__ double s_f[];  // NORM_TPB * ld
    const int64_t e0 = (int64_t)blockIdx.x * NORM_TPB;
    const int64_t ne = n_elems - e0 < NORM_TPB ? n_elems - e0 : NORM_TPB;
    const int64_t e = e0 + threadIdx.x;
    // the element's geometry first: its gathers overlap the staging below
    double adet = 0.0;
    if (e < n_elems) {
        int g[D + 1];
#pragma unroll
        for (int v = 0; v <= D; ++v) g[v] = __ldg(elems + e * (D + 1) + v);
        Geo<D> G;
        load_geo<D>(coords, g, G);
        adet = fabs(G.det);
    }
    stage_rows(fq + e0 * per, ne * per, per, ld, s_f);
    __syncthreads();
    if (e >= n_elems) return;
    const double* f = s_f + threadIdx.x * ld;
    double acc = 0.0;
    for (int q = 0; q < NQ; ++q) {
        double f2 = 0.0;
        for (int c = 0; c < nf; ++c) {
            const double v = f[q * nf + c];
            f2 += v * v;
        }
        acc += Q.w[q] * adet * f2;
    }
    per_elem[e] = acc;
}

template <int D>
__global__ void k_norm_elem(const double* __restrict__ coords, const int32_t* __restrict__ elems, int64_t n_elems,
                            const double* __restrict__ fq, int nf, double* __restrict__ per_elem) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    const Quad6& Q = quad(D);
    int g[D + 1];
#pragma unroll
    for (int v = 0; v <= D; ++v) g[v] = __ldg(elems + e * (D + 1) + v);
    Geo<D> G;
    load_geo<D>(coords, g, G);
    const double adet = fabs(G.det);
    const double* f = fq + e * Q.nq * nf;
    double acc = 0.0;
    for (int q = 0; q < Q.nq; ++q) {
        double f2 = 0.0;
        for (int c = 0; c < nf; ++c) {
            const double v = __ldg(f + q * nf + c);
            f2 += v * v;
        }
        acc += Q.w[q] * adet * f2;
    }
    per_elem[e] = acc;
}

// per element: ||E - v||^2_K and ||D E - D v||^2_K, v = sum_i c_i phi_i
template <class KT>
__global__ void k_field_error(const double* __restrict__ coords, const int32_t* __restrict__ elems, int64_t n_elems,
                              const int32_t* __restrict__ e2d, const double* __restrict__ coeffs,
                              const double* __restrict__ Eq, const double* __restrict__ Dq,
                              double* __restrict__ ev, double* __restrict__ ed) {
    constexpr int D = KT::D, NV = KT::NV, M = KT::M, ND = n_deriv<KT>();
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    const Quad6& Q = quad(D);
    int g[NV];
    load_g<KT>(elems, (int)e, g);
    Geo<D> G;
    load_geo<D>(coords, g, G);
    double c[M], s[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
        c[k] = __ldg(coeffs + __ldg(e2d + e * M + k));
        s[k] = sign_d<KT>(g, k);
    }
    double dv[ND];
#pragma unroll
    for (int r = 0; r < ND; ++r) dv[r] = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
        double d[ND];
        global_deriv<KT>(G, s[k], k, d);
#pragma unroll
        for (int r = 0; r < ND; ++r) dv[r] += c[k] * d[r];
    }
    const double adet = fabs(G.det);
    double a = 0.0, dd = 0.0;
    constexpr int NQ = D == 2 ? 12 : 24;
#pragma unroll 4
    for (int q = 0; q < NQ; ++q) {
        double v[D];
#pragma unroll
        for (int r = 0; r < D; ++r) v[r] = 0.0;
#pragma unroll
        for (int k = 0; k < M; ++k) {
            double phi[D];
            global_value<KT>(G, s[k], k, Q.l[q], phi);
#pragma unroll
            for (int r = 0; r < D; ++r) v[r] += c[k] * phi[r];
        }
        double ta = 0.0, td = 0.0;
#pragma unroll
        for (int r = 0; r < D; ++r) {
            const double x = __ldg(Eq + (e * NQ + q) * D + r) - v[r];
            ta += x * x;
        }
#pragma unroll
        for (int r = 0; r < ND; ++r) {
            const double x = __ldg(Dq + (e * NQ + q) * ND + r) - dv[r];
            td += x * x;
        }
        a += Q.w[q] * adet * ta;
        dd += Q.w[q] * adet * td;
    }
    ev[e] = a;
    ed[e] = dd;
}

// ---- fixed-order reductions ---------------------------------------------------------
constexpr int RED_TPB = 256;
constexpr int RED_PARTS = 1024;

// part p sums v[p*chunk, (p+1)*chunk) with a fixed shared-memory tree
__global__ void __launch_bounds__(RED_TPB) k_reduce_parts(const double* __restrict__ v, int64_t n, int64_t chunk,
                                                          double* __restrict__ part) {
    __shared__ double sm[RED_TPB];
    const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += RED_TPB) acc += v[i];
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int s = RED_TPB / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

// out[0] = sum of part[0..np) (fixed tree); optional finalize
__global__ void __launch_bounds__(RED_TPB) k_reduce_final(const double* __restrict__ part, int np,
                                                          double* __restrict__ out) {
    __shared__ double sm[RED_TPB];
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += RED_TPB) acc += part[i];
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int s = RED_TPB / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = sm[0];
}

efem_status reduce_fixed(const double* v, int64_t n, double* part, double* out, cudaStream_t s) {
    const int64_t chunk = std::max<int64_t>(RED_TPB, (n + RED_PARTS - 1) / RED_PARTS);
    const int np = (int)((n + chunk - 1) / chunk);
    if (np > 0) {
        k_reduce_parts<<<np, RED_TPB, 0, s>>>(v, n, chunk, part);
        EFEM_LAUNCH_CHECK();
    }
    k_reduce_final<<<1, RED_TPB, 0, s>>>(part, np, out);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

// ---- SpMV and CG ----------------------------------------------------------------------
// y = alpha K x + beta M x on the shared pattern (one thread per row)
__global__ void k_spmv(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ vk,
                       const double* __restrict__ vm, double alpha, double beta, int64_t n, const double* __restrict__ x,
                       double* __restrict__ y) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int j = __ldg(rp + i); j < __ldg(rp + i + 1); ++j)
        acc += (alpha * __ldg(vk + j) + beta * __ldg(vm + j)) * __ldg(x + __ldg(ci + j));
    y[i] = acc;
}

__global__ void k_diag(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ vk,
                       const double* __restrict__ vm, double alpha, double beta, int64_t n, double* __restrict__ dinv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double d = 0.0;
    for (int j = rp[i]; j < rp[i + 1]; ++j)
        if (ci[j] == i) d = alpha * vk[j] + beta * vm[j];
    dinv[i] = d != 0.0 ? 1.0 / d : 1.0;
}

// elementwise product into a scratch vector (then reduced in fixed order)
__global__ void k_mul(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* __restrict__ o) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) o[i] = a[i] * b[i];
}

// x += a p ; r -= a q ; z = dinv r ; t1 = r z ; t2 = r r    (a = sc[0] / sc[1])
__global__ void k_cg_update(const double* __restrict__ sc, const double* __restrict__ p, const double* __restrict__ q,
                            const double* __restrict__ dinv, int64_t n, double* __restrict__ x, double* __restrict__ r,
                            double* __restrict__ z, double* __restrict__ t1, double* __restrict__ t2) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double a = sc[0] / sc[1];
    x[i] += a * p[i];
    const double ri = r[i] - a * q[i];
    r[i] = ri;
    const double zi = dinv[i] * ri;
    z[i] = zi;
    t1[i] = ri * zi;
    t2[i] = ri * ri;
}

// p = z + (rz_new / rz_old) p ; then rz_old = rz_new


// ---- fused CG iteration: the dot products are reduced per CTA by the kernel
// that produces their terms (fixed shared-memory tree), then across CTAs by
// one fixed-order final pass -- 5 launches per iteration instead of 11.
__device__ __forceinline__ double cta_sum(double v, double* sm) {  // RED_TPB threads, fixed tree
    sm[threadIdx.x] = v;
    __syncthreads();
    for (int s = RED_TPB / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
        __syncthreads();
    }
    return sm[0];
}

// q = (alpha K + beta M) p and the CTA partial of p.q
__global__ void __launch_bounds__(RED_TPB) k_cg_spmv(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                     const double* __restrict__ vk, const double* __restrict__ vm,
                                                     double alpha, double beta, int64_t n,
                                                     const double* __restrict__ p, double* __restrict__ q,
                                                     double* __restrict__ part_pq) {
    __shared__ double sm[RED_TPB];
    const int64_t i = blockIdx.x * (int64_t)RED_TPB + threadIdx.x;
    double pq = 0.0;
    if (i < n) {
        double acc = 0.0;
        for (int j = __ldg(rp + i); j < __ldg(rp + i + 1); ++j)
            acc += (alpha * __ldg(vk + j) + beta * __ldg(vm + j)) * __ldg(p + __ldg(ci + j));
        q[i] = acc;
        pq = p[i] * acc;
    }
    const double t = cta_sum(pq, sm);
    if (threadIdx.x == 0) part_pq[blockIdx.x] = t;
}

// x += a p, r -= a q, z = D^-1 r (a = rz_old / pq) and the CTA partials of r.z, r.r
__global__ void __launch_bounds__(RED_TPB) k_cg_step(const double* __restrict__ sc, int o,
                                                     const double* __restrict__ p, const double* __restrict__ q,
                                                     const double* __restrict__ dinv, int64_t n, double* __restrict__ x,
                                                     double* __restrict__ r, double* __restrict__ z,
                                                     double* __restrict__ part_rz, double* __restrict__ part_rr) {
    __shared__ double sm[RED_TPB];
    const int64_t i = blockIdx.x * (int64_t)RED_TPB + threadIdx.x;
    double rz = 0.0, rr = 0.0;
    if (i < n) {
        const double a = sc[o] / sc[2];
        x[i] += a * p[i];
        const double ri = r[i] - a * q[i];
        r[i] = ri;
        const double zi = dinv[i] * ri;
        z[i] = zi;
        rz = ri * zi;
        rr = ri * ri;
    }
    const double t1 = cta_sum(rz, sm);
    __syncthreads();
    const double t2 = cta_sum(rr, sm);
    if (threadIdx.x == 0) {
        part_rz[blockIdx.x] = t1;
        part_rr[blockIdx.x] = t2;
    }
}

// out_a = sum part_a[0..np), out_b = sum part_b[0..np) (fixed trees; block 0 / 1)
__global__ void __launch_bounds__(RED_TPB) k_reduce_final2(const double* __restrict__ part_a,
                                                           const double* __restrict__ part_b, int np,
                                                           double* __restrict__ out_a, double* __restrict__ out_b) {
    __shared__ double sm[RED_TPB];
    const double* part = blockIdx.x == 0 ? part_a : part_b;
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += RED_TPB) acc += part[i];
    const double t = cta_sum(acc, sm);
    if (threadIdx.x == 0) (blockIdx.x == 0 ? out_a : out_b)[0] = t;
}

// p = z + (rz_new / rz_old) p
__global__ void k_cg_dir2(const double* __restrict__ sc, int o, const double* __restrict__ z, int64_t n,
                          double* __restrict__ p) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    p[i] = z[i] + (sc[1 - o] / sc[o]) * p[i];
}

}  // namespace

// ---- launchers ------------------------------------------------------------------------
int quad6_size(int dim) { return dim == 2 ? 12 : 24; }

efem_status quad6_host(int dim, double* l, double* w) {
    const Quad6 q = make_quad6(dim);
    for (int i = 0; i < 24; ++i) {
        for (int c = 0; c < 3; ++c) l[3 * i + c] = q.l[i][c];
        w[i] = q.w[i];
    }
    return EFEM_OK;
}

efem_status launch_quad_points(int dim, const double* coords, const int32_t* elems, int64_t n_elems, double* pts,
                               cudaStream_t s) {
    efem_status st;
    if ((st = ensure_quad()) != EFEM_OK) return st;
    const int64_t n = n_elems * quad6_size(dim);
    if (n == 0) return EFEM_OK;
    if (dim == 2)
        k_quad_points<2><<<grid_for(n_elems, QP_TPB), QP_TPB, QP_TPB * 25 * 8, s>>>(coords, elems, n_elems, pts);
    else {
        // 3D: 73 doubles per element -> 73 KB per CTA (opt-in; per device, so set at every call)
        EFEM_CUDA_TRY(cudaFuncSetAttribute(k_quad_points<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           QP_TPB * 73 * 8));
        k_quad_points<3><<<grid_for(n_elems, QP_TPB), QP_TPB, QP_TPB * 73 * 8, s>>>(coords, elems, n_elems, pts);
    }
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

// element contributions staged in the plan's bucket-key array (enumeration
// scratch, >= 8 bytes per instance, free after the symbolic pass)
template <class KT, int PAIR>
efem_status load_kt2(Plan& p, const double* fq, double* b, cudaStream_t s) {
    constexpr int TPB = 128;
    constexpr int NF = PAIR == 0 ? KT::D : n_deriv<KT>();
    constexpr int NQ = KT::D == 2 ? 12 : 24;
    constexpr size_t smem = (size_t)TPB * ((NQ * NF) | 1) * 8;
    // (the shared-memory opt-in is per device: set at every call)
    EFEM_CUDA_TRY(cudaFuncSetAttribute(k_load_elem<KT, PAIR, TPB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    double* loc = reinterpret_cast<double*>(p.bkey);
    k_load_elem<KT, PAIR, TPB><<<grid_for(p.n_elems, TPB), TPB, smem, s>>>(p.coords, p.elems, p.n_elems, fq, loc);
    EFEM_LAUNCH_CHECK();
    k_load_gather<KT><<<grid_for(p.n_dofs, 256), 256, 0, s>>>(p.inc_ptr, p.bucket, p.n_dofs, loc, b);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

template <class KT>
efem_status load_kt(Plan& p, int pairing, const double* fq, double* b, cudaStream_t s) {
    return pairing == 0 ? load_kt2<KT, 0>(p, fq, b, s) : load_kt2<KT, 1>(p, fq, b, s);
}

efem_status launch_load(Plan& p, int pairing, const double* fq, double* b, cudaStream_t s) {
    efem_status st;
    if ((st = ensure_quad()) != EFEM_OK) return st;
    if (p.n_dofs == 0) return EFEM_OK;
    if (p.dim == 2) return p.element == EFEM_RT0 ? load_kt<Kind<2, EFEM_RT0>>(p, pairing, fq, b, s)
                                                 : load_kt<Kind<2, EFEM_NED0>>(p, pairing, fq, b, s);
    return p.element == EFEM_RT0 ? load_kt<Kind<3, EFEM_RT0>>(p, pairing, fq, b, s)
                                 : load_kt<Kind<3, EFEM_NED0>>(p, pairing, fq, b, s);
}

size_t reduce_ws_bytes() { return (size_t)(RED_PARTS + 8) * sizeof(double); }

efem_status launch_norm_l2(int dim, const double* coords, const int32_t* elems, int64_t n_elems, const double* fq,
                           int nf, double* per_elem, double* total, double* part, cudaStream_t s) {
    efem_status st;
    if ((st = ensure_quad()) != EFEM_OK) return st;
    if (n_elems > 0) {
        const int per = quad6_size(dim) * nf;
        const size_t smem = (size_t)NORM_TPB * (per | 1) * 8;
        if (smem <= 96 * 1024) {  // staged (coalesced) reads of the point values
            // (the shared-memory opt-in is per device: set at every call)
            EFEM_CUDA_TRY(cudaFuncSetAttribute(dim == 2 ? (const void*)k_norm_elem_staged<2>
                                                        : (const void*)k_norm_elem_staged<3>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
            if (dim == 2)
                k_norm_elem_staged<2><<<grid_for(n_elems, NORM_TPB), NORM_TPB, smem, s>>>(coords, elems, n_elems, fq,
                                                                                           nf, per_elem);
            else
                k_norm_elem_staged<3><<<grid_for(n_elems, NORM_TPB), NORM_TPB, smem, s>>>(coords, elems, n_elems, fq,
                                                                                           nf, per_elem);
        } else if (dim == 2) {
            k_norm_elem<2><<<grid_for(n_elems, 128), 128, 0, s>>>(coords, elems, n_elems, fq, nf, per_elem);
        } else {
            k_norm_elem<3><<<grid_for(n_elems, 128), 128, 0, s>>>(coords, elems, n_elems, fq, nf, per_elem);
        }
        EFEM_LAUNCH_CHECK();
    }
    return reduce_fixed(per_elem, n_elems, part, total, s);
}

template <class KT>
efem_status field_error_kt(Plan& p, const double* coeffs, const double* Eq, const double* Dq, double* ev, double* ed,
                           cudaStream_t s) {
    k_field_error<KT><<<grid_for(p.n_elems, 128), 128, 0, s>>>(p.coords, p.elems, p.n_elems, p.e2d, coeffs, Eq, Dq,
                                                               ev, ed);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status launch_field_error(Plan& p, const double* coeffs, const double* Eq, const double* Dq, double* err2,
                               double* scratch, cudaStream_t s) {
    efem_status st;
    if ((st = ensure_quad()) != EFEM_OK) return st;
    double* ev = scratch;
    double* ed = scratch + p.n_elems;
    double* part = scratch + 2 * p.n_elems;
    if (p.n_elems > 0) {
        if (p.dim == 2)
            st = p.element == EFEM_RT0 ? field_error_kt<Kind<2, EFEM_RT0>>(p, coeffs, Eq, Dq, ev, ed, s)
                                       : field_error_kt<Kind<2, EFEM_NED0>>(p, coeffs, Eq, Dq, ev, ed, s);
        else
            st = p.element == EFEM_RT0 ? field_error_kt<Kind<3, EFEM_RT0>>(p, coeffs, Eq, Dq, ev, ed, s)
                                       : field_error_kt<Kind<3, EFEM_NED0>>(p, coeffs, Eq, Dq, ev, ed, s);
        if (st != EFEM_OK) return st;
    }
    if ((st = reduce_fixed(ev, p.n_elems, part, err2, s)) != EFEM_OK) return st;
    return reduce_fixed(ed, p.n_elems, part, err2 + 1, s);
}

efem_status launch_spmv(const efem_csr* A, double alpha, double beta, const double* x, double* y, cudaStream_t s) {
    if (A->n_rows == 0) return EFEM_OK;
    k_spmv<<<grid_for(A->n_rows, 256), 256, 0, s>>>(A->row_ptr, A->col_idx, A->vals_stiff, A->vals_mass, alpha, beta,
                                                    A->n_rows, x, y);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

size_t cg_ws_bytes(int64_t n) { return (size_t)(7 * n + RED_PARTS + 16) * sizeof(double) + 256; }

// Jacobi-preconditioned CG on A = alpha K + beta M (SPD for alpha, beta > 0).
// Device-side scalars; the host reads the residual every `check` iterations.
efem_status run_cg(const efem_csr* A, double alpha, double beta, const double* b, double* x, double rtol, int maxit,
                   int* iters, double* relres, void* ws, cudaStream_t s) {
    const int64_t n = A->n_rows;
    double* w = reinterpret_cast<double*>(ws);
    double *r = w, *z = w + n, *p = w + 2 * n, *q = w + 3 * n, *dinv = w + 4 * n, *t1 = w + 5 * n, *t2 = w + 6 * n;
    double* part = w + 7 * n;
    double* sc = part + RED_PARTS;  // [0] rz  [1] pq  [2] rz_new  [3] rr  [4] bb
    const unsigned g = grid_for(n, 256);
    efem_status st;
    *iters = 0;
    *relres = 0.0;
    if (n == 0) return EFEM_OK;
    k_diag<<<g, 256, 0, s>>>(A->row_ptr, A->col_idx, A->vals_stiff, A->vals_mass, alpha, beta, n, dinv);
    EFEM_LAUNCH_CHECK();
    // r = b - A x ; z = D^-1 r ; p = z ; rz
    if ((st = launch_spmv(A, alpha, beta, x, q, s)) != EFEM_OK) return st;
    {
        double h[2];
        // r = b - q via k_cg_update with a = 1: x untouched needs p = 0 -> do it directly
        cudaMemcpyAsync(r, b, n * 8, cudaMemcpyDeviceToDevice, s);
        k_mul<<<g, 256, 0, s>>>(b, b, n, t2);
        EFEM_LAUNCH_CHECK();
        if ((st = reduce_fixed(t2, n, part, sc + 4, s)) != EFEM_OK) return st;
        // r -= q
        EFEM_CUDA_TRY(cudaMemsetAsync(p, 0, n * 8, s));
        const double one_one[2] = {1.0, 1.0};
        EFEM_CUDA_TRY(cudaMemcpyAsync(sc, one_one, 16, cudaMemcpyHostToDevice, s));
        k_cg_update<<<g, 256, 0, s>>>(sc, p, q, dinv, n, x, r, z, t1, t2);  // a = 1, p = 0: x unchanged
        EFEM_LAUNCH_CHECK();
        if ((st = reduce_fixed(t1, n, part, sc + 0, s)) != EFEM_OK) return st;
        if ((st = reduce_fixed(t2, n, part, sc + 3, s)) != EFEM_OK) return st;
        EFEM_CUDA_TRY(cudaMemcpyAsync(p, z, n * 8, cudaMemcpyDeviceToDevice, s));
        EFEM_CUDA_TRY(cudaMemcpyAsync(h, sc + 3, 16, cudaMemcpyDeviceToHost, s));
        EFEM_CUDA_TRY(cudaStreamSynchronize(s));
        const double bn = std::sqrt(h[1]);
        *relres = bn > 0 ? std::sqrt(h[0]) / bn : 0.0;
        if (bn == 0.0 || *relres <= rtol) return EFEM_OK;
    }
    const int check = 20;
    // scalars: sc[0] / sc[1] rz (ping-pong: the iteration's old value at sc[o]),
    // sc[2] p.q, sc[3] r.r, sc[4] b.b; CTA partials in t1 / t2 (n >> #CTAs)
    const unsigned gr = grid_for(n, RED_TPB);
    double *part_a = t1, *part_b = t2;
    int o = 0;
    for (int it = 1; it <= maxit; ++it) {
        k_cg_spmv<<<gr, RED_TPB, 0, s>>>(A->row_ptr, A->col_idx, A->vals_stiff, A->vals_mass, alpha, beta, n, p, q,
                                          part_a);
        EFEM_LAUNCH_CHECK();
        k_reduce_final<<<1, RED_TPB, 0, s>>>(part_a, (int)gr, sc + 2);
        EFEM_LAUNCH_CHECK();
        k_cg_step<<<gr, RED_TPB, 0, s>>>(sc, o, p, q, dinv, n, x, r, z, part_a, part_b);
        EFEM_LAUNCH_CHECK();
        k_reduce_final2<<<2, RED_TPB, 0, s>>>(part_a, part_b, (int)gr, sc + (1 - o), sc + 3);
        EFEM_LAUNCH_CHECK();
        k_cg_dir2<<<g, 256, 0, s>>>(sc, o, z, n, p);
        EFEM_LAUNCH_CHECK();
        o = 1 - o;
        *iters = it;
        if (it % check == 0 || it == maxit) {
            double h[2];
            EFEM_CUDA_TRY(cudaMemcpyAsync(h, sc + 3, 16, cudaMemcpyDeviceToHost, s));
            EFEM_CUDA_TRY(cudaStreamSynchronize(s));
            *relres = std::sqrt(h[0] / h[1]);
            if (*relres <= rtol) break;
        }
    }
    return EFEM_OK;
}

}  // namespace efem
