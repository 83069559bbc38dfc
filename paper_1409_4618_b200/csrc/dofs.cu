// dofs.cu -- DOF enumeration and orientation (
// get_edges / get_faces / signs_edges / signs_faces of Sec. 3).
//
// Global DOF = edge (2D, 3D NE0) or face (3D RT0), numbered by the
// lexicographic rank of its ascending node tuple (reading C10).  Instead of a
// global radix sort of T*m keys, each entity is owned
// by its minimum node a:
//   1. node -> element incidence by a counting sort (atomic histogram + scan
//      + atomic scatter);
//   2. per node a: collect the entities of its incident elements whose minimum
//      node is a, sort/unique them in registers  -> count (pass 1) -> exclusive
//      scan gives ent_ptr[a], the id of a's first entity -> (pass 2) write
//      dofs2nodes rows and elems2dofs / signs of the entities a owns.
// Since ids are ent_ptr[a] + rank among a's entities, this equals the
// lexicographic rank of (a, b[, c]) over all entities: byte-identical to a
// sort + unique.
#include "efem_internal.cuh"

namespace efem {

__global__ void k_incidence_count(const int32_t* __restrict__ elems, int64_t n_entries, int64_t n_nodes,
                                  int32_t* __restrict__ cnt, WsHeader* hdr) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_entries) return;
    const int v = elems[i];
    if ((unsigned)v >= (unsigned long long)n_nodes) {
        atomicOr(&hdr->flags[F_INVALID_NODE], 1);
        return;
    }
    atomicAdd(&cnt[v], 1);
}

template <int NV>
__global__ void k_incidence_fill(const int32_t* __restrict__ elems, int64_t n_entries, int64_t n_nodes,
                                 const int32_t* __restrict__ n2e_ptr, int32_t* __restrict__ cnt,
                                 int32_t* __restrict__ n2e) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_entries) return;
    const int v = elems[i];
    if ((unsigned)v >= (unsigned long long)n_nodes) return;
    const int pos = n2e_ptr[v] + atomicSub(&cnt[v], 1) - 1;
    n2e[pos] = (int)(((i / NV) << 2) | (i % NV));
}

template <class KT>
__device__ __forceinline__ void load_elem(const int32_t* __restrict__ elems, int e, int (&g)[KT::NV]) {
    if constexpr (KT::NV == 4) {
        const int4 t = __ldg(reinterpret_cast<const int4*>(elems) + e);
        g[0] = t.x; g[1] = t.y; g[2] = t.z; g[3] = t.w;
    } else {
        const int32_t* p = elems + (int64_t)e * 3;
        g[0] = __ldg(p); g[1] = __ldg(p + 1); g[2] = __ldg(p + 2);
    }
}

// sorted insert with dedupe into a per-thread list; returns false on overflow
__device__ __forceinline__ bool insert_key(uint64_t* keys, int& nk, uint64_t key) {
    int j = nk;
    while (j > 0 && keys[j - 1] > key) --j;
    if (j > 0 && keys[j - 1] == key) return true;
    if (nk >= EFEM_MAX_NODE_ENTITIES) return false;
    for (int t = nk; t > j; --t) keys[t] = keys[t - 1];
    keys[j] = key;
    ++nk;
    return true;
}

// Sign data (2D rule PAPER.md:528, 3D readings C3/C5/C6):
// edges: +1 iff global(start) < global(end) (tangent runs low -> high);
// faces: s = -sgn(pi), pi the permutation listing the face's local vertices
// by ascending global id followed by the opposite vertex.  This equals
// sign(det B_K) * sign(nu . (x_a - x_opp)) with nu = (x_b-x_a) x (x_c-x_a),
// a<b<c, because det B_K cancels.
template <class KT>
__device__ __forceinline__ int local_sign(const int (&g)[KT::NV], int k) {
    if constexpr (KT::FACES) {
        // face k = vertices {0,1,2,3} \ {3-k} in ascending local order, then 3-k.
        // base parity of (f0,f1,f2,opp): k=0 (0,1,2,3) even, k=1 (0,1,3,2) odd,
        // k=2 (0,2,3,1) even, k=3 (1,2,3,0) odd.
        const int o = 3 - k;
        int f[3], t = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v)
            if (v != o) f[t++] = g[v];
        const int inv = (f[0] > f[1]) + (f[0] > f[2]) + (f[1] > f[2]);
        const int base_odd = k & 1;
        const int odd = (inv + base_odd) & 1;
        return odd ? 1 : -1;  // s = -sgn(pi)
    } else {
        return g[edge_start(KT::D, k)] < g[edge_end(KT::D, k)] ? 1 : -1;
    }
}

template <class KT, bool FILL>
__global__ void __launch_bounds__(128) k_node_entities(const int32_t* __restrict__ elems,
                                                       const int32_t* __restrict__ n2e_ptr,
                                                       const int32_t* __restrict__ n2e, int64_t n_nodes,
                                                       int32_t* __restrict__ ent_cnt,
                                                       const int32_t* __restrict__ ent_ptr,
                                                       int32_t* __restrict__ d2n, int32_t* __restrict__ e2d,
                                                       WsHeader* hdr) {
    const int64_t a64 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a64 >= n_nodes) return;
    const int a = (int)a64;
    const int beg = n2e_ptr[a], end = n2e_ptr[a + 1];
    uint64_t keys[EFEM_MAX_NODE_ENTITIES];
    int nk = 0;
    bool ok = true;
    for (int p = beg; p < end; ++p) {
        const int ent = __ldg(n2e + p);
        const int e = ent >> 2, lv = ent & 3;
        int g[KT::NV];
        load_elem<KT>(elems, e, g);
        if constexpr (!KT::FACES) {
#pragma unroll
            for (int u = 0; u < KT::NV; ++u)
                if (u != lv && g[u] > a) ok &= insert_key(keys, nk, (uint64_t)(uint32_t)g[u]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int w = u + 1; w < 4; ++w)
                    if (u != lv && w != lv && g[u] > a && g[w] > a) {
                        const uint32_t lo = min(g[u], g[w]), hi = max(g[u], g[w]);
                        ok &= insert_key(keys, nk, ((uint64_t)lo << 32) | hi);
                    }
        }
    }
    if (!ok) atomicOr(&hdr->flags[F_CAPACITY], 1);
    if constexpr (!FILL) {
        ent_cnt[a] = nk;
    } else {
        const int base = ent_ptr[a];
        for (int r = 0; r < nk; ++r) {
            int32_t* row = d2n + (int64_t)(base + r) * KT::EK;
            row[0] = a;
            if constexpr (KT::FACES) {
                row[1] = (int)(keys[r] >> 32);
                row[2] = (int)(keys[r] & 0xffffffffu);
            } else {
                row[1] = (int)keys[r];
            }
        }
        // elems2dofs / signs of the entities whose minimum node is a
        for (int p = beg; p < end; ++p) {
            const int ent = __ldg(n2e + p);
            const int e = ent >> 2, lv = ent & 3;
            int g[KT::NV];
            load_elem<KT>(elems, e, g);
#pragma unroll
            for (int k = 0; k < KT::M; ++k) {
                uint64_t key;
                bool mine;
                if constexpr (KT::FACES) {
                    const int o = 3 - k;
                    int f[3], t = 0;
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        if (v != o) f[t++] = v;
                    const bool has = (f[0] == lv) | (f[1] == lv) | (f[2] == lv);
                    int lo = INT_MAX, hi = -1, mn = INT_MAX;
#pragma unroll
                    for (int q = 0; q < 3; ++q)
                        if (f[q] != lv) {
                            lo = min(lo, g[f[q]]);
                            hi = max(hi, g[f[q]]);
                        }
#pragma unroll
                    for (int q = 0; q < 3; ++q) mn = min(mn, g[f[q]]);
                    mine = has && mn == a && lo > a;
                    key = ((uint64_t)(uint32_t)lo << 32) | (uint32_t)hi;
                } else {
                    const int s0 = edge_start(KT::D, k), s1 = edge_end(KT::D, k);
                    const int other = s0 == lv ? s1 : s0;
                    mine = (s0 == lv || s1 == lv) && g[other] > a;
                    key = (uint64_t)(uint32_t)g[other];
                }
                if (!mine) continue;
                int lo = 0, hi = nk - 1, r = -1;
                while (lo <= hi) {
                    const int mid = (lo + hi) >> 1;
                    if (keys[mid] == key) { r = mid; break; }
                    if (keys[mid] < key) lo = mid + 1; else hi = mid - 1;
                }
                if (r < 0) { atomicOr(&hdr->flags[F_CAPACITY], 1); continue; }
                e2d[(int64_t)e * KT::M + k] = base + r;
            }
        }
    }
}

template <class KT>
__global__ void k_signs(const int32_t* __restrict__ elems, int64_t n_elems, int8_t* __restrict__ sgn) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    int g[KT::NV];
    load_elem<KT>(elems, (int)e, g);
#pragma unroll
    for (int k = 0; k < KT::M; ++k) sgn[e * KT::M + k] = (int8_t)local_sign<KT>(g, k);
}

efem_status launch_signs(Plan& p, int8_t* out, cudaStream_t s) {
    if (p.n_elems == 0) return EFEM_OK;
    const int tpb = 256;
    const unsigned grid = grid_for(p.n_elems, tpb);
    if (p.dim == 2 && p.element == EFEM_RT0) k_signs<Kind<2, EFEM_RT0>><<<grid, tpb, 0, s>>>(p.elems, p.n_elems, out);
    else if (p.dim == 2) k_signs<Kind<2, EFEM_NED0>><<<grid, tpb, 0, s>>>(p.elems, p.n_elems, out);
    else if (p.element == EFEM_RT0) k_signs<Kind<3, EFEM_RT0>><<<grid, tpb, 0, s>>>(p.elems, p.n_elems, out);
    else k_signs<Kind<3, EFEM_NED0>><<<grid, tpb, 0, s>>>(p.elems, p.n_elems, out);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

// explicit launchers -----------------------------------------------------------------
template <class KT>
efem_status launch_entities(Plan& p, bool fill, cudaStream_t s) {
    const int tpb = 128;
    const unsigned grid = grid_for(p.n_nodes, tpb);
    if (!fill)
        k_node_entities<KT, false><<<grid, tpb, 0, s>>>(p.elems, p.n2e_ptr, p.n2e, p.n_nodes, p.ent_cnt, nullptr,
                                                        nullptr, nullptr, p.hdr);
    else
        k_node_entities<KT, true><<<grid, tpb, 0, s>>>(p.elems, p.n2e_ptr, p.n2e, p.n_nodes, nullptr, p.ent_ptr,
                                                       p.d2n, p.e2d, p.hdr);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status launch_incidence(Plan& p, cudaStream_t s) {
    const int64_t n_entries = p.n_elems * p.nv;
    const int tpb = 256;
    if (n_entries == 0) return EFEM_OK;
    k_incidence_count<<<grid_for(n_entries, tpb), tpb, 0, s>>>(p.elems, n_entries, p.n_nodes, p.cnt, p.hdr);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status launch_incidence_fill(Plan& p, cudaStream_t s) {
    const int64_t n_entries = p.n_elems * p.nv;
    const int tpb = 256;
    if (n_entries == 0) return EFEM_OK;
    if (p.nv == 3)
        k_incidence_fill<3><<<grid_for(n_entries, tpb), tpb, 0, s>>>(p.elems, n_entries, p.n_nodes, p.n2e_ptr,
                                                                     p.cnt, p.n2e);
    else
        k_incidence_fill<4><<<grid_for(n_entries, tpb), tpb, 0, s>>>(p.elems, n_entries, p.n_nodes, p.n2e_ptr,
                                                                     p.cnt, p.n2e);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status launch_entities_any(Plan& p, bool fill, cudaStream_t s) {
    if (p.n_nodes == 0) return EFEM_OK;
    if (p.dim == 2) return p.element == EFEM_RT0 ? launch_entities<Kind<2, EFEM_RT0>>(p, fill, s)
                                                 : launch_entities<Kind<2, EFEM_NED0>>(p, fill, s);
    return p.element == EFEM_RT0 ? launch_entities<Kind<3, EFEM_RT0>>(p, fill, s)
                                 : launch_entities<Kind<3, EFEM_NED0>>(p, fill, s);
}

}  // namespace efem
