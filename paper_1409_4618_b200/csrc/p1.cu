// p1.cu -- linear nodal (P1) elements for the majorant example (SURVEY.md
// §8(f) f3; "The approximation v was calculated with linear
// nodal finite elements"): the node -> element incidence by a counting sort,
// row structure = sorted distinct vertices of a node's elements, the
// Laplacian stiffness K_ab = |K| grad l_a . grad l_b and mass
// M_ab = |K| (1 + d_ab) / ((d+1)(d+2)) summed per row in ascending element
// order, the load sum_K sum_q w |det| f l_a, grad v at the quadrature points,
// and symmetric Dirichlet elimination.  Not the hot path; product code only.
#include <atomic>
#include <cub/cub.cuh>

#include <new>

#include "efem_internal.cuh"

namespace efem {

constexpr int P1_ROW_CAP = 64;   // elements per node held per thread
constexpr int P1_W_CAP = 64;     // distinct neighbours (incl. the node) per row

struct P1Plan {
    int dim = 0;
    int64_t n_nodes = 0, n_elems = 0;
    const double* coords = nullptr;
    const int32_t* elems = nullptr;
    char* ws = nullptr;
    size_t ws_need = 0, cub_bytes = 0;
    int32_t *cnt = nullptr, *node_ptr = nullptr, *inc = nullptr, *rowlen = nullptr, *row_ptr = nullptr;
    int* flags = nullptr;  // [0] capacity exceeded, [1] degenerate
    void* cub_tmp = nullptr;
    int64_t nnz = 0;
    bool symbolic = false;
};

// quadrature of integrate.cu (degree 6) -- declared there
int quad6_size(int dim);
efem_status quad6_host(int dim, double* l /* 24 x 3 */, double* w /* 24 */);

namespace {

size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

template <int D>
__device__ __forceinline__ double p1_grads(const double* __restrict__ coords, const int32_t* g, double (&gl)[D + 1][D]) {
    double X[D + 1][D];
#pragma unroll
    for (int v = 0; v <= D; ++v)
#pragma unroll
        for (int c = 0; c < D; ++c) X[v][c] = __ldg(coords + (int64_t)g[v] * D + c);
    double B[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) B[r][c] = X[c + 1][r] - X[0][r];
    double det;
    if constexpr (D == 2) {
        det = B[0][0] * B[1][1] - B[0][1] * B[1][0];
        // rows of B^{-1}: grad l_1, grad l_2
        gl[1][0] = B[1][1] / det;
        gl[1][1] = -B[0][1] / det;
        gl[2][0] = -B[1][0] / det;
        gl[2][1] = B[0][0] / det;
    } else {
        double cof[3][3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int r1 = (r + 1) % 3, r2 = (r + 2) % 3, c1 = (c + 1) % 3, c2 = (c + 2) % 3;
                cof[r][c] = B[r1][c1] * B[r2][c2] - B[r1][c2] * B[r2][c1];
            }
        det = B[0][0] * cof[0][0] + B[0][1] * cof[0][1] + B[0][2] * cof[0][2];
        // B^{-1}[i][r] = cof[r][i] / det
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int r = 0; r < 3; ++r) gl[i + 1][r] = cof[r][i] / det;
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
        double s = 0.0;
#pragma unroll
        for (int i = 1; i <= D; ++i) s += gl[i][r];
        gl[0][r] = -s;
    }
    return det;
}

template <int D, bool FILL>
__global__ void k_p1_bucket(const int32_t* __restrict__ elems, int64_t n_elems, int64_t n_nodes,
                            int32_t* __restrict__ cnt, const int32_t* __restrict__ node_ptr,
                            int32_t* __restrict__ inc, int* flags) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
#pragma unroll
    for (int v = 0; v <= D; ++v) {
        const int a = __ldg(elems + e * (D + 1) + v);
        if ((unsigned)a >= (unsigned long long)n_nodes) {
            if (!FILL) atomicOr(&flags[2], 1);
            continue;
        }
        if constexpr (!FILL) {
            atomicAdd(&cnt[a], 1);
        } else {
            const int pos = atomicSub(&cnt[a], 1) - 1;  // counts return to zero
            inc[__ldg(node_ptr + a) + pos] = (int)e;
        }
    }
}

// per node: sort its elements ascending, count distinct vertices (the row)
template <int D>
__global__ void k_p1_rows(const int32_t* __restrict__ elems, const int32_t* __restrict__ node_ptr,
                          int32_t* __restrict__ inc, int64_t n_nodes, int32_t* __restrict__ rowlen, int* flags) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n_nodes) return;
    const int b0 = node_ptr[a], n = node_ptr[a + 1] - b0;
    int32_t* L = inc + b0;
    for (int j = 1; j < n; ++j) {  // insertion sort (small lists)
        const int v = L[j];
        int q = j;
        while (q > 0 && L[q - 1] > v) {
            L[q] = L[q - 1];
            --q;
        }
        L[q] = v;
    }
    int W[P1_W_CAP];
    int nw = 0;
    bool over = false;
    W[nw++] = (int)a;
    for (int j = 0; j < n; ++j)
        for (int v = 0; v <= D; ++v) {
            const int x = __ldg(elems + (int64_t)L[j] * (D + 1) + v);
            bool seen = false;
            for (int u = 0; u < nw; ++u) seen |= W[u] == x;
            if (seen) continue;
            if (nw == P1_W_CAP) {
                over = true;
                continue;
            }
            W[nw++] = x;
        }
    if (over || n > P1_ROW_CAP) atomicOr(&flags[0], 1);
    rowlen[a] = nw;
}

template <int D>
__global__ void k_p1_numeric(const double* __restrict__ coords, const int32_t* __restrict__ elems,
                             const int32_t* __restrict__ node_ptr, const int32_t* __restrict__ inc,
                             const int32_t* __restrict__ row_ptr, int64_t n_nodes, int32_t* __restrict__ col_idx,
                             double* __restrict__ vm, double* __restrict__ vk, int32_t* __restrict__ rp_out,
                             int* flags) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n_nodes) return;
    const int b0 = node_ptr[a], n = min(node_ptr[a + 1] - b0, P1_ROW_CAP);
    const int r0 = row_ptr[a], rl = row_ptr[a + 1] - r0;
    rp_out[a] = r0;
    if (a == n_nodes - 1) rp_out[n_nodes] = r0 + rl;
    if (rl > P1_W_CAP) return;  // flagged by k_p1_rows
    int W[P1_W_CAP];
    double am[P1_W_CAP], ak[P1_W_CAP];
    int nw = 0;
    W[nw++] = (int)a;
    for (int j = 0; j < n; ++j)
        for (int v = 0; v <= D; ++v) {
            const int x = __ldg(elems + (int64_t)inc[b0 + j] * (D + 1) + v);
            int q = nw;
            bool seen = false;
            for (int u = 0; u < nw; ++u) seen |= W[u] == x;
            if (seen || nw == P1_W_CAP) continue;
            while (q > 0 && W[q - 1] > x) {  // keep W sorted
                W[q] = W[q - 1];
                --q;
            }
            W[q] = x;
            ++nw;
        }
    for (int u = 0; u < nw; ++u) am[u] = ak[u] = 0.0;
    const double cm = D == 2 ? 1.0 / 12.0 : 1.0 / 20.0;  // 1 / ((d+1)(d+2))
    for (int j = 0; j < n; ++j) {
        const int e = inc[b0 + j];
        int g[D + 1];
#pragma unroll
        for (int v = 0; v <= D; ++v) g[v] = __ldg(elems + (int64_t)e * (D + 1) + v);
        double gl[D + 1][D];
        const double det = p1_grads<D>(coords, g, gl);
        if (!(det != 0.0) || !isfinite(det)) atomicOr(&flags[1], 1);
        const double vol = fabs(det) / (D == 2 ? 2.0 : 6.0);
        int la = 0;
#pragma unroll
        for (int v = 1; v <= D; ++v) la = g[v] == a ? v : la;
        double ga[D];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double t = gl[0][r];
#pragma unroll
            for (int v = 1; v <= D; ++v) t = la == v ? gl[v][r] : t;
            ga[r] = t;
        }
#pragma unroll
        for (int v = 0; v <= D; ++v) {
            int lo = 0, hi = nw - 1;  // position of g[v] in W
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (W[mid] < g[v]) lo = mid + 1; else hi = mid;
            }
            double dot = 0.0;
#pragma unroll
            for (int r = 0; r < D; ++r) dot += ga[r] * gl[v][r];
            ak[lo] += vol * dot;
            am[lo] += vol * (v == la ? 2.0 : 1.0) * cm;
        }
    }
    for (int u = 0; u < nw; ++u) {
        col_idx[r0 + u] = W[u];
        if (vm) vm[r0 + u] = am[u];
        if (vk) vk[r0 + u] = ak[u];
    }
}

struct P1Quad {
    double l[24][3];
    double w[24];
    int nq;
};
__constant__ P1Quad c_p1q[2];
std::atomic<bool> g_p1q[64];  // per device (__constant__ memory is per device)

efem_status ensure_p1q() {
    int dev = 0;
    EFEM_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 64 && g_p1q[dev].load(std::memory_order_acquire)) return EFEM_OK;
    P1Quad q[2]{};
    for (int d = 2; d <= 3; ++d) {
        efem_status st = quad6_host(d, &q[d - 2].l[0][0], q[d - 2].w);
        if (st != EFEM_OK) return st;
        q[d - 2].nq = quad6_size(d);
    }
    EFEM_CUDA_TRY(cudaMemcpyToSymbol(c_p1q, q, sizeof(q)));
    if (dev < 64) g_p1q[dev].store(true, std::memory_order_release);
    return EFEM_OK;
}

template <int D>
__global__ void k_p1_load(const double* __restrict__ coords, const int32_t* __restrict__ elems,
                          const int32_t* __restrict__ node_ptr, const int32_t* __restrict__ inc, int64_t n_nodes,
                          const double* __restrict__ fq, double* __restrict__ b) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n_nodes) return;
    const P1Quad& Q = c_p1q[D - 2];
    const int b0 = node_ptr[a], n = node_ptr[a + 1] - b0;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {  // ascending element order (sorted by k_p1_rows)
        const int e = inc[b0 + j];
        int g[D + 1];
#pragma unroll
        for (int v = 0; v <= D; ++v) g[v] = __ldg(elems + (int64_t)e * (D + 1) + v);
        double gl[D + 1][D];
        const double adet = fabs(p1_grads<D>(coords, g, gl));
        int la = 0;
#pragma unroll
        for (int v = 1; v <= D; ++v) la = g[v] == a ? v : la;
        double loc = 0.0;
        for (int q = 0; q < Q.nq; ++q) {
            double lam = 1.0;
#pragma unroll
            for (int i = 0; i < D; ++i) lam -= Q.l[q][i];
#pragma unroll
            for (int i = 0; i < D; ++i) lam = la == i + 1 ? Q.l[q][i] : lam;
            loc += Q.w[q] * adet * __ldg(fq + (int64_t)e * Q.nq + q) * lam;
        }
        acc += loc;
    }
    b[a] = acc;
}

template <int D>
__global__ void k_p1_grad_q(const double* __restrict__ coords, const int32_t* __restrict__ elems, int64_t n_elems,
                            int nq, const double* __restrict__ v, double* __restrict__ out) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    int g[D + 1];
#pragma unroll
    for (int k = 0; k < D + 1; ++k) g[k] = __ldg(elems + e * (D + 1) + k);
    double gl[D + 1][D];
    p1_grads<D>(coords, g, gl);
    double gv[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k <= D; ++k) s += __ldg(v + g[k]) * gl[k][r];
        gv[r] = s;
    }
    for (int q = 0; q < nq; ++q)
#pragma unroll
        for (int r = 0; r < D; ++r) out[(e * nq + q) * D + r] = gv[r];
}

// symmetric Dirichlet elimination: masked rows / columns zeroed, K diagonal 1
__global__ void k_dirichlet(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            double* __restrict__ vk, double* __restrict__ vm, int64_t n,
                            const uint8_t* __restrict__ mask, double* __restrict__ b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool mi = mask[i] != 0;
    for (int j = rp[i]; j < rp[i + 1]; ++j) {
        const int c = ci[j];
        if (mi || mask[c]) {
            if (vk) vk[j] = (mi && c == i) ? 1.0 : 0.0;
            if (vm) vm[j] = 0.0;
        }
    }
    if (mi && b) b[i] = 0.0;
}

}  // namespace
}  // namespace efem

using namespace efem;

extern "C" {

efem_status efem_p1_plan_create(efem_p1_plan* plan, const efem_mesh* mesh, size_t* ws_bytes) {
    if (!plan || !mesh || !ws_bytes || (mesh->dim != 2 && mesh->dim != 3) || mesh->n_nodes < 0 ||
        mesh->n_elems < 0 || (mesh->n_elems > 0 && (!mesh->coords || !mesh->elems))) {
        set_error("efem_p1_plan_create: bad mesh");
        return EFEM_EINVAL;
    }
    if ((mesh->n_elems * (mesh->dim + 1)) >= (1ll << 31) || mesh->n_nodes >= (1ll << 31) - 1) {
        set_error("efem_p1_plan_create: mesh too large for int32 indexing");
        return EFEM_EOVERFLOW;
    }
    P1Plan* p = new (std::nothrow) P1Plan;
    if (!p) return EFEM_ENOMEM;
    p->dim = mesh->dim;
    p->n_nodes = mesh->n_nodes;
    p->n_elems = mesh->n_elems;
    p->coords = mesh->coords;
    p->elems = mesh->elems;
    size_t cb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cb, (const int32_t*)nullptr, (int32_t*)nullptr, (int)(p->n_nodes + 1));
    p->cub_bytes = cb;
    const size_t N1 = (size_t)p->n_nodes + 1, I = (size_t)p->n_elems * (p->dim + 1);
    p->ws_need = a256(64) + 4 * a256(N1 * 4) + a256(I * 4 + 4) + a256(cb);
    *ws_bytes = p->ws_need;
    *plan = reinterpret_cast<efem_p1_plan>(p);
    return EFEM_OK;
}

efem_status efem_p1_plan_set_workspace(efem_p1_plan plan, void* ws, size_t ws_bytes) {
    P1Plan* p = reinterpret_cast<P1Plan*>(plan);
    if (!p || !ws || ws_bytes < p->ws_need || (reinterpret_cast<uintptr_t>(ws) & 255)) {
        set_error("efem_p1_plan_set_workspace: workspace NULL, too small or not 256-byte aligned");
        return EFEM_EWORKSPACE;
    }
    char* b = static_cast<char*>(ws);
    const size_t N1 = (size_t)p->n_nodes + 1, I = (size_t)p->n_elems * (p->dim + 1);
    p->ws = b;
    p->flags = reinterpret_cast<int*>(b);
    b += a256(64);
    p->cnt = reinterpret_cast<int32_t*>(b);
    b += a256(N1 * 4);
    p->node_ptr = reinterpret_cast<int32_t*>(b);
    b += a256(N1 * 4);
    p->rowlen = reinterpret_cast<int32_t*>(b);
    b += a256(N1 * 4);
    p->row_ptr = reinterpret_cast<int32_t*>(b);
    b += a256(N1 * 4);
    p->inc = reinterpret_cast<int32_t*>(b);
    b += a256(I * 4 + 4);
    p->cub_tmp = b;
    EFEM_CUDA_TRY(cudaMemset(p->cnt, 0, N1 * 4));
    EFEM_CUDA_TRY(cudaMemset(p->rowlen, 0, N1 * 4));
    p->symbolic = false;
    return EFEM_OK;
}

efem_status efem_p1_plan_destroy(efem_p1_plan plan) {
    delete reinterpret_cast<P1Plan*>(plan);
    return EFEM_OK;
}

efem_status efem_p1_symbolic(efem_p1_plan plan, int64_t* n_rows, int64_t* nnz, efem_stream_t stream) {
    P1Plan* p = reinterpret_cast<P1Plan*>(plan);
    if (!p || !p->ws) {
        set_error("efem_p1_symbolic: plan without workspace");
        return EFEM_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t N = p->n_nodes, T = p->n_elems;
    EFEM_CUDA_TRY(cudaMemsetAsync(p->flags, 0, 64, s));
    if (T > 0) {
        if (p->dim == 2) k_p1_bucket<2, false><<<grid_for(T, 256), 256, 0, s>>>(p->elems, T, N, p->cnt, nullptr, nullptr, p->flags);
        else k_p1_bucket<3, false><<<grid_for(T, 256), 256, 0, s>>>(p->elems, T, N, p->cnt, nullptr, nullptr, p->flags);
        EFEM_LAUNCH_CHECK();
    }
    size_t cb = p->cub_bytes;
    EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p->cub_tmp, cb, p->cnt, p->node_ptr, (int)(N + 1), s));
    if (T > 0) {
        if (p->dim == 2) k_p1_bucket<2, true><<<grid_for(T, 256), 256, 0, s>>>(p->elems, T, N, p->cnt, p->node_ptr, p->inc, p->flags);
        else k_p1_bucket<3, true><<<grid_for(T, 256), 256, 0, s>>>(p->elems, T, N, p->cnt, p->node_ptr, p->inc, p->flags);
        EFEM_LAUNCH_CHECK();
    }
    if (N > 0) {
        if (p->dim == 2) k_p1_rows<2><<<grid_for(N, 128), 128, 0, s>>>(p->elems, p->node_ptr, p->inc, N, p->rowlen, p->flags);
        else k_p1_rows<3><<<grid_for(N, 128), 128, 0, s>>>(p->elems, p->node_ptr, p->inc, N, p->rowlen, p->flags);
        EFEM_LAUNCH_CHECK();
    }
    cb = p->cub_bytes;
    EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p->cub_tmp, cb, p->rowlen, p->row_ptr, (int)(N + 1), s));
    int h[4];
    int32_t tot = 0;
    EFEM_CUDA_TRY(cudaMemcpyAsync(h, p->flags, 16, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaMemcpyAsync(&tot, p->row_ptr + N, 4, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    if (h[2]) {
        set_error("efem_p1_symbolic: an element references a node id outside [0, n_nodes)");
        return EFEM_EINVAL;
    }
    if (h[0]) {
        set_error("efem_p1_symbolic: a node touches more than 64 elements or 63 neighbours");
        return EFEM_ECAPACITY;
    }
    p->nnz = tot;
    p->symbolic = true;
    if (n_rows) *n_rows = N;
    if (nnz) *nnz = tot;
    return EFEM_OK;
}

efem_status efem_p1_numeric(efem_p1_plan plan, efem_csr* out, efem_stream_t stream) {
    P1Plan* p = reinterpret_cast<P1Plan*>(plan);
    if (!p || !p->symbolic || !out || out->n_rows != p->n_nodes || out->nnz != p->nnz || !out->row_ptr ||
        (p->nnz > 0 && !out->col_idx)) {
        set_error("efem_p1_numeric: call efem_p1_symbolic first; out sizes must match");
        return EFEM_ESTATE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t N = p->n_nodes;
    if (N == 0) {
        EFEM_CUDA_TRY(cudaMemsetAsync(out->row_ptr, 0, 4, s));
        return EFEM_OK;
    }
    if (p->dim == 2)
        k_p1_numeric<2><<<grid_for(N, 128), 128, 0, s>>>(p->coords, p->elems, p->node_ptr, p->inc, p->row_ptr, N,
                                                         out->col_idx, out->vals_mass, out->vals_stiff, out->row_ptr,
                                                         p->flags);
    else
        k_p1_numeric<3><<<grid_for(N, 128), 128, 0, s>>>(p->coords, p->elems, p->node_ptr, p->inc, p->row_ptr, N,
                                                         out->col_idx, out->vals_mass, out->vals_stiff, out->row_ptr,
                                                         p->flags);
    EFEM_LAUNCH_CHECK();
    int h[2];
    EFEM_CUDA_TRY(cudaMemcpyAsync(h, p->flags, 8, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    if (h[1]) {
        set_error("efem_p1_numeric: degenerate element");
        return EFEM_EDEGENERATE;
    }
    return EFEM_OK;
}

efem_status efem_p1_load(efem_p1_plan plan, const double* fq, double* b, efem_stream_t stream) {
    P1Plan* p = reinterpret_cast<P1Plan*>(plan);
    if (!p || !p->symbolic || (p->n_nodes > 0 && (!fq || !b))) {
        set_error("efem_p1_load: call efem_p1_symbolic first; arrays non-NULL");
        return EFEM_ESTATE;
    }
    efem_status st = ensure_p1q();
    if (st != EFEM_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t N = p->n_nodes;
    if (N == 0) return EFEM_OK;
    if (p->dim == 2) k_p1_load<2><<<grid_for(N, 128), 128, 0, s>>>(p->coords, p->elems, p->node_ptr, p->inc, N, fq, b);
    else k_p1_load<3><<<grid_for(N, 128), 128, 0, s>>>(p->coords, p->elems, p->node_ptr, p->inc, N, fq, b);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status efem_p1_gradient(const efem_mesh* mesh, const double* v, double* grad_q, efem_stream_t stream) {
    if (!mesh || (mesh->dim != 2 && mesh->dim != 3) || (mesh->n_elems > 0 && (!v || !grad_q))) {
        set_error("efem_p1_gradient: bad arguments");
        return EFEM_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t T = mesh->n_elems;
    if (T == 0) return EFEM_OK;
    const int nq = quad6_size(mesh->dim);
    if (mesh->dim == 2) k_p1_grad_q<2><<<grid_for(T, 128), 128, 0, s>>>(mesh->coords, mesh->elems, T, nq, v, grad_q);
    else k_p1_grad_q<3><<<grid_for(T, 128), 128, 0, s>>>(mesh->coords, mesh->elems, T, nq, v, grad_q);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status efem_dirichlet(efem_csr* A, const uint8_t* mask, double* b, efem_stream_t stream) {
    if (!A || A->n_rows < 0 || (A->n_rows > 0 && (!mask || !A->row_ptr || !A->col_idx))) {
        set_error("efem_dirichlet: bad arguments");
        return EFEM_EINVAL;
    }
    if (A->n_rows == 0) return EFEM_OK;
    k_dirichlet<<<grid_for(A->n_rows, 256), 256, 0, (cudaStream_t)stream>>>(A->row_ptr, A->col_idx, A->vals_stiff,
                                                                            A->vals_mass, A->n_rows, mask, b);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

}  // extern "C"
