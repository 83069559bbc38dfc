// part.cu -- row-owned partitioned assembly for multi-GPU runs (SURVEY.md
// §8(e)).
//
// Rank r owns the rows of the entities whose minimum node lies in its node
// range [lo, hi) (DOF ids are lexicographic in node ids, so this is a
// contiguous block of global rows).  It assembles them from a sub-mesh: the
// elements touching the nodes of the elements touching [lo, hi) (two hops),
// so every entity that appears in an owned row has its minimum node's full
// star locally and gets the same rank among that node's entities as in the
// global mesh.  The only exchange is an allgather of the per-node entity
// counts of the owned ranges (global DOF offsets) and of the per-rank CSR
// entry counts (row offsets): owner computes, no matrix values cross ranks.
#include <cub/cub.cuh>

#include <algorithm>

#include "efem_internal.cuh"

namespace efem {
namespace {

template <int NV>
__global__ void k_mark_touch(const int32_t* __restrict__ elems, int64_t n_elems, const int8_t* __restrict__ node_in,
                             int64_t lo, int64_t hi, int8_t* __restrict__ node_out, int8_t* __restrict__ elem_out) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    int g[NV];
    bool hit = false;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        g[v] = __ldg(elems + e * NV + v);
        hit |= node_in ? node_in[g[v]] != 0 : (g[v] >= lo && g[v] < hi);
    }
    if (!hit) return;
    if (elem_out) elem_out[e] = 1;
#pragma unroll
    for (int v = 0; v < NV; ++v) node_out[g[v]] = 1;
}

__global__ void k_i8_to_i32(const int8_t* __restrict__ in, int32_t* __restrict__ out, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
    if (i == n) out[i] = 0;
}

template <int NV>
__global__ void k_fill_sub(const double* __restrict__ coords, const int32_t* __restrict__ elems, int64_t n_elems,
                           int64_t n_nodes, int dim, const int32_t* __restrict__ elem_pos,
                           const int32_t* __restrict__ node_pos, double* __restrict__ sub_coords,
                           int32_t* __restrict__ sub_elems, int32_t* __restrict__ sub2global) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n_elems && elem_pos[i + 1] != elem_pos[i]) {
        const int64_t o = elem_pos[i];
#pragma unroll
        for (int v = 0; v < NV; ++v) sub_elems[o * NV + v] = node_pos[elems[i * NV + v]];
    }
    if (i < n_nodes && node_pos[i + 1] != node_pos[i]) {
        const int64_t o = node_pos[i];
        sub2global[o] = (int32_t)i;
        for (int c = 0; c < dim; ++c) sub_coords[o * dim + c] = coords[i * dim + c];
    }
}

struct PartWs {
    int8_t* node1;
    int8_t* node2;
    int8_t* elem2;
    int32_t* node_pos;
    int32_t* elem_pos;
    int32_t* node_tmp;
    int32_t* elem_tmp;
    void* cub;
    size_t cub_bytes;
};

size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

PartWs part_layout(char* b, int64_t N, int64_t T, size_t cub_bytes, size_t* total) {
    PartWs w{};
    size_t off = 0;
    auto take = [&](size_t n) {
        size_t o = off;
        off += a256(n);
        return b ? b + o : nullptr;
    };
    w.node1 = (int8_t*)take(N);
    w.node2 = (int8_t*)take(N);
    w.elem2 = (int8_t*)take(T);
    w.node_pos = (int32_t*)take((N + 1) * 4);
    w.elem_pos = (int32_t*)take((T + 1) * 4);
    w.node_tmp = (int32_t*)take((N + 1) * 4);
    w.elem_tmp = (int32_t*)take((T + 1) * 4);
    w.cub = take(cub_bytes);
    w.cub_bytes = cub_bytes;
    *total = off;
    return w;
}

size_t part_cub_bytes(int64_t N, int64_t T) {
    size_t bytes = 0;
    const int64_t n = (N > T ? N : T) + 1;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
    return bytes;
}

__global__ void k_lower_bound(const int32_t* __restrict__ sorted, int64_t n, int64_t key0, int64_t key1,
                              int64_t* __restrict__ out) {
    // out[0] = first index with sorted >= key0, out[1] = first with sorted >= key1
    if (threadIdx.x > 1 || blockIdx.x) return;
    const int64_t key = threadIdx.x == 0 ? key0 : key1;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sorted[mid] < key) lo = mid + 1; else hi = mid;
    }
    out[threadIdx.x] = lo;
}

__global__ void k_owned_counts(const int32_t* __restrict__ ent_ptr, const int32_t* __restrict__ sub2global,
                               int64_t l0, int64_t l1, int64_t lo, int32_t* __restrict__ owned_cnt) {
    const int64_t u = l0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u >= l1) return;
    owned_cnt[sub2global[u] - lo] = ent_ptr[u + 1] - ent_ptr[u];
}

// per local node u: global id of its first entity minus the local one
__global__ void k_node_shift(const int32_t* __restrict__ ent_ptr, const int32_t* __restrict__ sub2global,
                             const int32_t* __restrict__ global_ent_ptr, int64_t n_nodes, int32_t* __restrict__ shift) {
    const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u < n_nodes) shift[u] = global_ent_ptr[sub2global[u]] - ent_ptr[u];
}

// a local DOF d of minimum node u has global id d + shift[u]
template <class KT>
__global__ void k_globalize(const int32_t* __restrict__ elems, int64_t n_elems, const int32_t* __restrict__ e2d,
                            const int32_t* __restrict__ shift, int32_t* __restrict__ e2d_global) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    int g[KT::NV];
#pragma unroll
    for (int v = 0; v < KT::NV; ++v) g[v] = elems[e * KT::NV + v];
#pragma unroll
    for (int k = 0; k < KT::M; ++k) {
        int u;
        if constexpr (KT::FACES) {
            u = INT_MAX;
#pragma unroll
            for (int v = 0; v < 4; ++v)
                if (v != 3 - k) u = min(u, g[v]);
        } else {
            u = min(g[edge_start(KT::D, k)], g[edge_end(KT::D, k)]);
        }
        e2d_global[e * KT::M + k] = e2d[e * KT::M + k] + __ldg(shift + u);
    }
}


// Row window of a bound partition (one thread): local rows [ent_ptr[l0],
// ent_ptr[l1]) and their CSR entries in the sub-mesh's local numbering.
__global__ void k_part_window(const int32_t* __restrict__ ent_ptr, const int32_t* __restrict__ inc_ptr,
                              const int32_t* __restrict__ row_ptr, int64_t l0, int64_t l1, int c,
                              long long* __restrict__ win) {
    if (threadIdx.x || blockIdx.x) return;
    if (l1 <= l0) {  // no owned node in the sub-mesh: an empty window
        win[0] = win[1] = win[2] = win[3] = 0;
        return;
    }
    const long long r0 = ent_ptr[l0], r1 = ent_ptr[l1];
    auto start = [&](long long r) -> long long { return row_ptr ? row_ptr[r] : r + (long long)c * inc_ptr[r]; };
    const long long z0 = start(r0), z1 = start(r1);
    win[0] = r0;
    win[1] = r1 - r0;
    win[2] = z0;
    win[3] = z1 - z0;
}

__global__ void k_empty_window_check(WsHeader* hdr) {  // a zero-capacity slice fits only an empty window
    if (threadIdx.x || blockIdx.x) return;
    if (hdr->win[1] > 0 || hdr->win[3] > 0) atomicOr(&hdr->flags[F_CAPACITY], 1);
}

__global__ void k_part_first_row(const int32_t* __restrict__ global_ent_ptr, int64_t lo, long long* __restrict__ win) {
    if (threadIdx.x || blockIdx.x) return;
    win[4] = global_ent_ptr[lo];
}

// O(interface) globalisation: global first DOF id per SUB-MESH node
__global__ void k_node_shift_sub(const int32_t* __restrict__ ent_ptr, const int32_t* __restrict__ sub_first,
                                 int64_t n_nodes, int32_t* __restrict__ shift) {
    const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u < n_nodes) shift[u] = sub_first[u] - ent_ptr[u];
}

__global__ void k_part_first_row_sub(const int32_t* __restrict__ sub_first, int64_t l0, int64_t l1,
                                     long long* __restrict__ win) {
    if (threadIdx.x || blockIdx.x) return;
    win[4] = l1 > l0 ? sub_first[l0] : 0;
}

// first ids of the owned nodes: local exclusive prefix + the totals of the
// ranks before `rank` (totals: device, one int per rank)
__global__ void k_add_offset(int32_t* __restrict__ first, int64_t n, const int32_t* __restrict__ totals, int rank) {
    __shared__ int off;
    if (threadIdx.x == 0) {
        int o = 0;
        for (int r = 0; r < rank; ++r) o += totals[r];
        off = o;
    }
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        first[i] += off;
}

__global__ void k_index_gather(int32_t* __restrict__ dst, const int32_t* __restrict__ src,
                               const int32_t* __restrict__ idx, int64_t n, int32_t bias) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i] + bias];
}

__global__ void k_index_scatter(int32_t* __restrict__ dst, const int32_t* __restrict__ idx,
                                const int32_t* __restrict__ src, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[idx[i]] = src[i];
}

}  // namespace

efem_status launch_rows_any(Plan& p, unsigned forms, efem_csr* out, const RowWindow& w, cudaStream_t s);
efem_status launch_enumerate(Plan& p, cudaStream_t s);
bool row_ptr_stored(const Plan& p);

}  // namespace efem

using namespace efem;

extern "C" {

efem_status efem_partition(const efem_mesh* full, int64_t node_lo, int64_t node_hi, void* ws, size_t* ws_bytes,
                           int64_t* n_sub_nodes, int64_t* n_sub_elems, double* sub_coords, int32_t* sub_elems,
                           int32_t* sub2global, efem_stream_t stream) {
    if (!full || !ws_bytes || (full->dim != 2 && full->dim != 3) || node_lo < 0 || node_hi < node_lo ||
        node_hi > full->n_nodes) {
        set_error("efem_partition: bad arguments");
        return EFEM_EINVAL;
    }
    const int64_t N = full->n_nodes, T = full->n_elems;
    const int nv = full->dim + 1;
    size_t total = 0;
    const size_t cb = part_cub_bytes(N, T);
    part_layout(nullptr, N, T, cb, &total);
    if (!ws) {
        *ws_bytes = total;
        return EFEM_OK;
    }
    if (*ws_bytes < total || !n_sub_nodes || !n_sub_elems) {
        set_error("efem_partition: workspace too small or NULL size outputs");
        return EFEM_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    PartWs w = part_layout((char*)ws, N, T, cb, &total);
    const int tpb = 256;
    if (!sub_coords) {  // phase 1: marks and sizes
        EFEM_CUDA_TRY(cudaMemsetAsync(w.node1, 0, N, s));
        EFEM_CUDA_TRY(cudaMemsetAsync(w.node2, 0, N, s));
        EFEM_CUDA_TRY(cudaMemsetAsync(w.elem2, 0, T, s));
        if (T > 0) {
            if (nv == 3) {
                k_mark_touch<3><<<grid_for(T, tpb), tpb, 0, s>>>(full->elems, T, nullptr, node_lo, node_hi, w.node1,
                                                                 nullptr);
                k_mark_touch<3><<<grid_for(T, tpb), tpb, 0, s>>>(full->elems, T, w.node1, 0, 0, w.node2, w.elem2);
            } else {
                k_mark_touch<4><<<grid_for(T, tpb), tpb, 0, s>>>(full->elems, T, nullptr, node_lo, node_hi, w.node1,
                                                                 nullptr);
                k_mark_touch<4><<<grid_for(T, tpb), tpb, 0, s>>>(full->elems, T, w.node1, 0, 0, w.node2, w.elem2);
            }
            EFEM_LAUNCH_CHECK();
        }
        k_i8_to_i32<<<grid_for(N + 1, tpb), tpb, 0, s>>>(w.node2, w.node_tmp, N);
        k_i8_to_i32<<<grid_for(T + 1, tpb), tpb, 0, s>>>(w.elem2, w.elem_tmp, T);
        EFEM_LAUNCH_CHECK();
        size_t b1 = w.cub_bytes;
        EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.cub, b1, w.node_tmp, w.node_pos, (int)(N + 1), s));
        b1 = w.cub_bytes;
        EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.cub, b1, w.elem_tmp, w.elem_pos, (int)(T + 1), s));
        int32_t h[2];
        EFEM_CUDA_TRY(cudaMemcpyAsync(&h[0], w.node_pos + N, 4, cudaMemcpyDeviceToHost, s));
        EFEM_CUDA_TRY(cudaMemcpyAsync(&h[1], w.elem_pos + T, 4, cudaMemcpyDeviceToHost, s));
        EFEM_CUDA_TRY(cudaStreamSynchronize(s));
        *n_sub_nodes = h[0];
        *n_sub_elems = h[1];
        return EFEM_OK;
    }
    // phase 2: fill (the workspace must still hold phase 1's scans)
    if (!sub_elems || !sub2global) {
        set_error("efem_partition: NULL output arrays");
        return EFEM_EINVAL;
    }
    const int64_t n = N > T ? N : T;
    if (n > 0) {
        if (nv == 3)
            k_fill_sub<3><<<grid_for(n, tpb), tpb, 0, s>>>(full->coords, full->elems, T, N, full->dim, w.elem_pos,
                                                           w.node_pos, sub_coords, sub_elems, sub2global);
        else
            k_fill_sub<4><<<grid_for(n, tpb), tpb, 0, s>>>(full->coords, full->elems, T, N, full->dim, w.elem_pos,
                                                           w.node_pos, sub_coords, sub_elems, sub2global);
        EFEM_LAUNCH_CHECK();
    }
    return EFEM_OK;
}

efem_status efem_part_counts(efem_plan plan, const int32_t* sub2global, int64_t node_lo, int64_t node_hi,
                             int32_t* owned_cnt, int64_t* info, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !p->symbolic || !sub2global || !owned_cnt || !info || node_hi < node_lo) {
        set_error("efem_part_counts: needs a plan after efem_assemble_symbolic and non-NULL arrays");
        return EFEM_ESTATE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    {
        const efem_status e = ensure_enumerated(*p, s);  // (2D symbolic runs the fan pipeline)
        if (e != EFEM_OK) return e;
    }
    if (node_hi > node_lo) EFEM_CUDA_TRY(cudaMemsetAsync(owned_cnt, 0, (node_hi - node_lo) * 4, s));
    int64_t* d = reinterpret_cast<int64_t*>(p->d_totals);  // scratch: totals already read back
    k_lower_bound<<<1, 32, 0, s>>>(sub2global, p->n_nodes, node_lo, node_hi, d);
    EFEM_LAUNCH_CHECK();
    int64_t lr[2];
    EFEM_CUDA_TRY(cudaMemcpyAsync(lr, d, 16, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    if (lr[1] > lr[0]) {
        k_owned_counts<<<grid_for(lr[1] - lr[0], 256), 256, 0, s>>>(p->ent_ptr, sub2global, lr[0], lr[1], node_lo,
                                                                    owned_cnt);
        EFEM_LAUNCH_CHECK();
    }
    int32_t rows[2];
    int64_t nz[2];
    EFEM_CUDA_TRY(cudaMemcpyAsync(&rows[0], p->ent_ptr + lr[0], 4, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaMemcpyAsync(&rows[1], p->ent_ptr + lr[1], 4, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    efem_status st;
    if ((st = row_start_host(*p, rows[0], &nz[0], s)) != EFEM_OK) return st;
    if ((st = row_start_host(*p, rows[1], &nz[1], s)) != EFEM_OK) return st;
    info[0] = rows[0];          // first owned local row
    info[1] = rows[1] - rows[0];  // owned rows
    info[2] = nz[0];            // local CSR offset of the first owned row
    info[3] = nz[1] - nz[0];    // owned CSR entries
    return EFEM_OK;
}

efem_status efem_part_scan(const int32_t* global_cnt, int64_t n, int32_t* global_ent_ptr, void* ws, size_t* ws_bytes,
                           efem_stream_t stream) {
    if (!ws_bytes || n < 0) {
        set_error("efem_part_scan: bad arguments");
        return EFEM_EINVAL;
    }
    size_t need = 0, need2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, (const int32_t*)nullptr, (int32_t*)nullptr, (int)(n + 1));
    cub::DeviceScan::InclusiveSum(nullptr, need2, (const int32_t*)nullptr, (int32_t*)nullptr, (int)(n + 1));
    if (need2 > need) need = need2;
    need += 256 + (size_t)(n + 1) * 4;
    if (!ws) {
        *ws_bytes = need;
        return EFEM_OK;
    }
    if (*ws_bytes < need || !global_cnt || !global_ent_ptr) {
        set_error("efem_part_scan: workspace too small or NULL arrays");
        return EFEM_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    // global_ent_ptr[0] = 0, [i + 1] = inclusive sum of the first i + 1 counts
    char* cub_ws = reinterpret_cast<char*>(ws) + a256((size_t)(n + 1) * 4);
    size_t cb = need - 256 - (size_t)(n + 1) * 4;
    EFEM_CUDA_TRY(cudaMemsetAsync(global_ent_ptr, 0, 4, s));
    if (n > 0) {
        EFEM_CUDA_TRY(cub::DeviceScan::InclusiveSum(cub_ws, cb, global_cnt, global_ent_ptr + 1, (int)n, s));
        count_launch(2);
    }
    return EFEM_OK;
}

efem_status efem_part_globalize(efem_plan plan, const int32_t* sub2global, const int32_t* global_ent_ptr,
                                int32_t* e2d_global, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !(p->symbolic || (p->part_bound && p->async_pending)) || !sub2global || !global_ent_ptr || !e2d_global) {
        set_error("efem_part_globalize: needs a plan after efem_assemble_symbolic (or efem_part_enumerate_async) "
                  "and non-NULL arrays");
        return EFEM_ESTATE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (!p->async_pending) {
        const efem_status e = ensure_enumerated(*p, s);
        if (e != EFEM_OK) return e;
    }
    if (p->n_elems == 0) {
        if (p->part_bound) {
            k_part_first_row<<<1, 32, 0, s>>>(global_ent_ptr, p->part_lo, p->hdr->win);
            EFEM_LAUNCH_CHECK();
        }
        return EFEM_OK;
    }
    // (ent_cnt is scratch between enumerations: it holds the shifts here)
    int32_t* shift = p->ent_cnt;
    k_node_shift<<<grid_for(p->n_nodes, 256), 256, 0, s>>>(p->ent_ptr, sub2global, global_ent_ptr, p->n_nodes, shift);
    EFEM_LAUNCH_CHECK();
    const unsigned grid = grid_for(p->n_elems, 256);
    if (p->dim == 2 && p->element == EFEM_RT0)
        k_globalize<Kind<2, EFEM_RT0>><<<grid, 256, 0, s>>>(p->elems, p->n_elems, p->e2d, shift, e2d_global);
    else if (p->dim == 2)
        k_globalize<Kind<2, EFEM_NED0>><<<grid, 256, 0, s>>>(p->elems, p->n_elems, p->e2d, shift, e2d_global);
    else if (p->element == EFEM_RT0)
        k_globalize<Kind<3, EFEM_RT0>><<<grid, 256, 0, s>>>(p->elems, p->n_elems, p->e2d, shift, e2d_global);
    else
        k_globalize<Kind<3, EFEM_NED0>><<<grid, 256, 0, s>>>(p->elems, p->n_elems, p->e2d, shift, e2d_global);
    EFEM_LAUNCH_CHECK();
    if (p->part_bound) {  // the window's global first row, for efem_part_numeric_async
        k_part_first_row<<<1, 32, 0, s>>>(global_ent_ptr, p->part_lo, p->hdr->win);
        EFEM_LAUNCH_CHECK();
    }
    return EFEM_OK;
}

efem_status efem_part_numeric(efem_plan plan, unsigned forms, const int64_t* info, int64_t global_first_row,
                              const int32_t* e2d_global, efem_csr* slice, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !p->symbolic || !info || !e2d_global || !slice || slice->n_rows != info[1] || slice->nnz != info[3] ||
        (forms & ~7u)) {
        set_error("efem_part_numeric: slice sizes must match efem_part_counts");
        return EFEM_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    {
        const efem_status e = ensure_enumerated(*p, s);
        if (e != EFEM_OK) return e;
    }
    if (info[1] == 0) {  // the row kernels write row_ptr; an empty slice still needs its 0
        if (forms & EFEM_PATTERN) EFEM_CUDA_TRY(cudaMemsetAsync(slice->row_ptr, 0, 4, s));
        return EFEM_OK;
    }
    RowWindow w;
    w.row0 = info[0];
    w.n_rows = info[1];
    w.own_base = (int)global_first_row;
    w.out_base = (int)info[2];
    w.e2d = e2d_global;
    return launch_rows_any(*p, forms, slice, w, s);
}

// ---- bound partitions: the asynchronous step -----------------------------------
efem_status efem_part_bind(efem_plan plan, const int32_t* sub2global, int64_t node_lo, int64_t node_hi,
                           efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !p->ws || !sub2global || node_lo < 0 || node_hi < node_lo) {
        set_error("efem_part_bind: needs a plan with workspace, sub2global and 0 <= node_lo <= node_hi");
        return EFEM_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    int64_t* d = reinterpret_cast<int64_t*>(&p->hdr->win[0]);
    k_lower_bound<<<1, 32, 0, s>>>(sub2global, p->n_nodes, node_lo, node_hi, d);
    EFEM_LAUNCH_CHECK();
    int64_t lr[2];
    EFEM_CUDA_TRY(cudaMemcpyAsync(lr, d, 16, cudaMemcpyDeviceToHost, s));
    EFEM_CUDA_TRY(cudaStreamSynchronize(s));
    p->part_lo = node_lo;
    p->part_hi = node_hi;
    p->part_l0 = lr[0];
    p->part_l1 = lr[1];
    p->part_sub2global = sub2global;
    p->part_bound = true;
    if (p->g_part) {
        cudaGraphExecDestroy(p->g_part);
        p->g_part = nullptr;
    }
    return EFEM_OK;
}

efem_status efem_part_enumerate_async(efem_plan plan, int32_t* owned_cnt, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !p->ws || !p->part_bound || !owned_cnt) {
        set_error("efem_part_enumerate_async: needs a bound plan (efem_part_bind) and owned_cnt");
        return EFEM_ESTATE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    p->enumerated = p->symbolic = false;
    p->async_pending = true;
    p->async_fan = false;
    auto enqueue = [&](cudaStream_t q) -> efem_status {
        efem_status e = launch_enumerate(*p, q);
        if (e != EFEM_OK) return e;
        const int64_t width = p->part_hi - p->part_lo;
        if (width > 0) EFEM_CUDA_TRY(cudaMemsetAsync(owned_cnt, 0, width * 4, q));
        if (p->part_l1 > p->part_l0) {
            k_owned_counts<<<grid_for(p->part_l1 - p->part_l0, 256), 256, 0, q>>>(
                p->ent_ptr, p->part_sub2global, p->part_l0, p->part_l1, p->part_lo, owned_cnt);
            EFEM_LAUNCH_CHECK();
        }
        k_part_window<<<1, 32, 0, q>>>(p->ent_ptr, p->inc_ptr, row_ptr_stored(*p) ? p->row_ptr : nullptr,
                                        p->part_l0, p->part_l1, p->m - 1, p->hdr->win);
        EFEM_LAUNCH_CHECK();
        return EFEM_OK;
    };
    if (p->g_part && p->part_key != owned_cnt) {
        cudaGraphExecDestroy(p->g_part);
        p->g_part = nullptr;
    }
    if (!p->g_part && !p->graph_failed && !p->want_d2n && !debug_sync()) {
        bool ok = p->gstream != nullptr;
        if (!ok) {
            ok = cudaStreamCreateWithFlags(&p->gstream, cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming) == cudaSuccess;
        }
        cudaGraph_t graph = nullptr;
        if (ok && cudaStreamBeginCapture(p->gstream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            const int64_t l0 = efem_launch_count();
            const efem_status e = enqueue(p->gstream);
            const cudaError_t ee = cudaStreamEndCapture(p->gstream, &graph);
            p->part_launches = efem_launch_count() - l0;
            count_launch(-(int)p->part_launches);  // counted at replay
            if (e == EFEM_OK && ee == cudaSuccess && cudaGraphInstantiate(&p->g_part, graph, 0) == cudaSuccess)
                p->part_key = owned_cnt;
            else
                p->g_part = nullptr;
            if (graph) cudaGraphDestroy(graph);
        }
        cudaGetLastError();
    }
    if (p->g_part) {
        // (a graph captured on the plan's stream replays on the caller's)
        EFEM_CUDA_TRY(cudaGraphLaunch(p->g_part, s));
        count_launch((int)p->part_launches);
        return EFEM_OK;
    }
    return enqueue(s);
}

efem_status efem_part_numeric_async(efem_plan plan, unsigned forms, const int32_t* e2d_global, efem_csr* slice,
                                    efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !p->part_bound || !p->async_pending || !e2d_global || !slice || slice->n_rows < 0 ||
        slice->nnz < 0 || !slice->row_ptr || (forms & ~7u) ||
        (slice->nnz > 0 && (!slice->col_idx || ((forms & EFEM_MASS) && !slice->vals_mass) ||
                            ((forms & EFEM_STIFF) && !slice->vals_stiff)))) {
        set_error("efem_part_numeric_async: needs efem_part_enumerate_async + efem_part_globalize first, and a "
                  "slice with capacities and arrays");
        return EFEM_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (slice->n_rows == 0) {  // capacity 0: only an empty window fits
        if (forms & EFEM_PATTERN) EFEM_CUDA_TRY(cudaMemsetAsync(slice->row_ptr, 0, 4, s));
        k_empty_window_check<<<1, 32, 0, s>>>(p->hdr);
        EFEM_LAUNCH_CHECK();
        return EFEM_OK;
    }
    RowWindow w;
    w.row0 = 0;
    w.n_rows = slice->n_rows;
    w.e2d = e2d_global;
    w.cap_nnz = slice->nnz;
    w.win = p->hdr->win;
    return launch_rows_any(*p, forms, slice, w, s);
}

efem_status efem_part_window(efem_plan plan, int64_t* window_dev, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !p->part_bound || !window_dev) {
        set_error("efem_part_window: needs a bound plan and a device array of 5 int64");
        return EFEM_EINVAL;
    }
    EFEM_CUDA_TRY(cudaMemcpyAsync(window_dev, p->hdr->win, 5 * 8, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return EFEM_OK;
}

// ---- O(interface) globalisation of the owner-computes partition ------------------------
efem_status efem_part_add_offset(int32_t* first, int64_t n, const int32_t* totals, int rank, efem_stream_t stream) {
    if ((n > 0 && !first) || !totals || rank < 0) {
        set_error("efem_part_add_offset: NULL array or negative rank");
        return EFEM_EINVAL;
    }
    const unsigned grid = (unsigned)std::min<int64_t>(grid_for(std::max<int64_t>(n, 1), 256), 1024);
    k_add_offset<<<grid, 256, 0, (cudaStream_t)stream>>>(first, n, totals, rank);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status efem_index_gather(int32_t* dst, const int32_t* src, const int32_t* idx, int64_t n, int32_t bias,
                              efem_stream_t stream) {
    if (n < 0 || (n > 0 && (!dst || !src || !idx))) {
        set_error("efem_index_gather: NULL array");
        return EFEM_EINVAL;
    }
    if (n == 0) return EFEM_OK;
    k_index_gather<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(dst, src, idx, n, bias);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status efem_index_scatter(int32_t* dst, const int32_t* idx, const int32_t* src, int64_t n, efem_stream_t stream) {
    if (n < 0 || (n > 0 && (!dst || !src || !idx))) {
        set_error("efem_index_scatter: NULL array");
        return EFEM_EINVAL;
    }
    if (n == 0) return EFEM_OK;
    k_index_scatter<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(dst, idx, src, n);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status efem_part_globalize_sub(efem_plan plan, const int32_t* sub_first, int64_t l0, int64_t l1,
                                    int32_t* e2d_global, efem_stream_t stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p || !(p->symbolic || (p->part_bound && p->async_pending)) || !sub_first || !e2d_global) {
        set_error("efem_part_globalize_sub: needs a plan after efem_assemble_symbolic (or "
                  "efem_part_enumerate_async) and non-NULL arrays");
        return EFEM_ESTATE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (!p->async_pending) {
        const efem_status e = ensure_enumerated(*p, s);
        if (e != EFEM_OK) return e;
    }
    if (p->n_elems > 0) {
        int32_t* shift = p->ent_cnt;  // (scratch between enumerations)
        k_node_shift_sub<<<grid_for(p->n_nodes, 256), 256, 0, s>>>(p->ent_ptr, sub_first, p->n_nodes, shift);
        EFEM_LAUNCH_CHECK();
        const unsigned grid = grid_for(p->n_elems, 256);
        if (p->dim == 2 && p->element == EFEM_RT0)
            k_globalize<Kind<2, EFEM_RT0>><<<grid, 256, 0, s>>>(p->elems, p->n_elems, p->e2d, shift, e2d_global);
        else if (p->dim == 2)
            k_globalize<Kind<2, EFEM_NED0>><<<grid, 256, 0, s>>>(p->elems, p->n_elems, p->e2d, shift, e2d_global);
        else if (p->element == EFEM_RT0)
            k_globalize<Kind<3, EFEM_RT0>><<<grid, 256, 0, s>>>(p->elems, p->n_elems, p->e2d, shift, e2d_global);
        else
            k_globalize<Kind<3, EFEM_NED0>><<<grid, 256, 0, s>>>(p->elems, p->n_elems, p->e2d, shift, e2d_global);
        EFEM_LAUNCH_CHECK();
    }
    if (p->part_bound) {
        k_part_first_row_sub<<<1, 32, 0, s>>>(sub_first, l0, l1, p->hdr->win);
        EFEM_LAUNCH_CHECK();
    }
    return EFEM_OK;
}

}  // extern "C"
