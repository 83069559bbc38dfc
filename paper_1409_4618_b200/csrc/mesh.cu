// mesh.cu -- seeded structured mesh generator (input generator; DESIGN.md
// "Inputs").  Bit-identical to the oracle's ora_build_mesh because both
// implement the same recipe with separately rounded IEEE operations
// (__ddiv_rn / __dmul_rn / __dadd_rn here, -ffp-contract=off there).
#include "efem_internal.cuh"

namespace efem {
namespace {

__device__ __forceinline__ uint64_t counter_hash(uint64_t seed, uint64_t idx) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (idx + 1ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double grid_coord(int i, int n, bool interior, double alpha, uint64_t seed,
                                             uint64_t hidx) {
    const double x = __ddiv_rn((double)i, (double)n);
    if (!interior) return x;
    const double u = __dmul_rn((double)(counter_hash(seed, hidx) >> 11), 0x1.0p-53);
    double t = __dmul_rn(2.0, u);
    t = __dadd_rn(t, -1.0);
    const double h = __ddiv_rn(alpha, (double)n);
    return __dadd_rn(x, __dmul_rn(t, h));
}

__global__ void k_coords(int dim, int n, double alpha, uint64_t seed, int64_t n_nodes, double* __restrict__ coords) {
    const int64_t node = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (node >= n_nodes) return;
    const int64_t n1 = n + 1;
    const int i = (int)(node % n1);
    const int j = (int)((node / n1) % n1);
    const int k = dim == 3 ? (int)(node / (n1 * n1)) : 0;
    bool in = i > 0 && i < n && j > 0 && j < n;
    if (dim == 3) in = in && k > 0 && k < n;
    const int idx[3] = {i, j, k};
    for (int c = 0; c < dim; ++c)
        coords[node * dim + c] = grid_coord(idx[c], n, in, alpha, seed, (uint64_t)node * dim + c);
}

__global__ void k_elems2d(int n, int32_t* __restrict__ elems) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= (int64_t)n * n) return;
    const int n1 = n + 1;
    const int i = (int)(c % n), j = (int)(c / n);
    const int32_t v00 = i + n1 * j, v10 = v00 + 1, v01 = v00 + n1, v11 = v01 + 1;
    int32_t* e = elems + 6 * c;
    e[0] = v00; e[1] = v10; e[2] = v11;
    e[3] = v00; e[4] = v11; e[5] = v01;
}

__global__ void k_elems3d(int n, int32_t* __restrict__ elems) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= (int64_t)n * n * n) return;
    const int64_t n1 = n + 1;
    const int i = (int)(c % n), j = (int)((c / n) % n), k = (int)(c / ((int64_t)n * n));
    const int64_t stride[3] = {1, n1, n1 * n1};
    const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const int64_t v0 = i + stride[1] * j + stride[2] * k;
#pragma unroll
    for (int p = 0; p < 6; ++p) {
        int4 t;
        int64_t v = v0;
        t.x = (int)v;
        v += stride[perm[p][0]];
        t.y = (int)v;
        v += stride[perm[p][1]];
        t.z = (int)v;
        v += stride[perm[p][2]];
        t.w = (int)v;
        reinterpret_cast<int4*>(elems)[6 * c + p] = t;
    }
}

// L-shape (0,1)^2 minus (1/2,1)^2 on the m x m grid (m even, h = m/2): cells
// (i, j) with i >= h and j >= h removed, nodes (i, j) with i > h and j > h
// removed, both numbered row-major over what remains (reading L1).
__device__ __forceinline__ int64_t lnode(int i, int j, int m) {
    const int h = m / 2;
    return j <= h ? (int64_t)j * (m + 1) + i : (int64_t)(h + 1) * (m + 1) + (int64_t)(j - h - 1) * (h + 1) + i;
}

__global__ void k_lshape_coords(int m, double alpha, uint64_t seed, int64_t n_nodes, double* __restrict__ coords) {
    const int64_t node = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (node >= n_nodes) return;
    const int h = m / 2;
    const int64_t lower = (int64_t)(h + 1) * (m + 1);
    int i, j;
    if (node < lower) {
        j = (int)(node / (m + 1));
        i = (int)(node % (m + 1));
    } else {
        j = h + 1 + (int)((node - lower) / (h + 1));
        i = (int)((node - lower) % (h + 1));
    }
    const bool in = i > 0 && i < m && j > 0 && j < m && !(i >= h && j >= h);
    coords[2 * node + 0] = grid_coord(i, m, in, alpha, seed, (uint64_t)node * 2 + 0);
    coords[2 * node + 1] = grid_coord(j, m, in, alpha, seed, (uint64_t)node * 2 + 1);
}

__global__ void k_lshape_elems(int m, int64_t n_cells, int32_t* __restrict__ elems) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    const int h = m / 2;
    const int64_t lower = (int64_t)h * m;
    int i, j;
    if (c < lower) {
        j = (int)(c / m);
        i = (int)(c % m);
    } else {
        j = h + (int)((c - lower) / h);
        i = (int)((c - lower) % h);
    }
    const int32_t v00 = (int32_t)lnode(i, j, m), v10 = (int32_t)lnode(i + 1, j, m);
    const int32_t v01 = (int32_t)lnode(i, j + 1, m), v11 = (int32_t)lnode(i + 1, j + 1, m);
    int32_t* e = elems + 6 * c;
    e[0] = v00; e[1] = v10; e[2] = v11;
    e[3] = v00; e[4] = v11; e[5] = v01;
}

}  // namespace

efem_status launch_build_lshape(int m, double alpha, uint64_t seed, double* coords, int32_t* elems, cudaStream_t s) {
    const int h = m / 2;
    const int64_t N = (int64_t)(h + 1) * (m + 1) + (int64_t)(m - h) * (h + 1);
    const int64_t C = (int64_t)h * m + (int64_t)(m - h) * h;
    k_lshape_coords<<<grid_for(N, 256), 256, 0, s>>>(m, alpha, seed, N, coords);
    EFEM_LAUNCH_CHECK();
    k_lshape_elems<<<grid_for(C, 256), 256, 0, s>>>(m, C, elems);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status launch_build_mesh(int dim, int n, double alpha, uint64_t seed, double* coords, int32_t* elems,
                              cudaStream_t s) {
    const int64_t n1 = n + 1;
    const int64_t N = dim == 2 ? n1 * n1 : n1 * n1 * n1;
    const int tpb = 256;
    k_coords<<<grid_for(N, tpb), tpb, 0, s>>>(dim, n, alpha, seed, N, coords);
    EFEM_LAUNCH_CHECK();
    if (dim == 2) {
        k_elems2d<<<grid_for((int64_t)n * n, tpb), tpb, 0, s>>>(n, elems);
    } else {
        k_elems3d<<<grid_for((int64_t)n * n * n, tpb), tpb, 0, s>>>(n, elems);
    }
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

}  // namespace efem
