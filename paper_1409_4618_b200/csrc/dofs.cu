// dofs.cu -- DOF enumeration, orientation and CSR row lengths
// (get_edges / get_faces / signs_edges /
// signs_faces of Sec. 3; PAPER.md:696 for the sparse pattern).
//
// Global DOF = edge (2D, 3D NE0) or face (3D RT0), numbered by the
// lexicographic rank of its ascending node tuple (reading C10).  Instead of a
// global radix sort of T*m keys, every (element,
// local entity) INSTANCE is bucketed by the entity's minimum node a with one
// counting sort:
//   k_bucket<count>  instances per minimum node          (warp-aggregated atomics)
//   CUB scan         -> bucket_ptr
//   k_bucket<fill>   scatter (e << 3 | k) into the buckets
//   k_node_entities  per node: sort its bucket by (other nodes, element id);
//                    runs of equal keys are its entities, numbered
//                    ent_ptr[a] + run index, which IS the lexicographic rank.
//                    The sorted bucket is the entity -> element incidence
//                    (ascending element id per entity), inc_ptr = run starts.
//                    Row lengths (exact, no union needed):
//                      2D edges / 3D faces: 1 + (m-1) t   (two elements share
//                        at most one entity of that kind),
//                      3D edges: 1 + 2 L + t   (L distinct link vertices c give
//                        edges a-c and b-c; each tet adds one link edge),
//                    t = elements containing the entity.  Node offsets of both
//                    entities and row entries come from one decoupled
//                    look-back scan inside the same kernel.
#include <cub/cub.cuh>

#include "efem_internal.cuh"
#include "scan.cuh"

namespace efem {

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

// minimum node of local entity k: edges (start, end), faces the three
// vertices other than 3-k
template <class KT>
__device__ __forceinline__ int entity_min_node(const int (&g)[KT::NV], int k) {
    if constexpr (KT::FACES) {
        const int o = 3 - k;
        int mn = INT_MAX;
#pragma unroll
        for (int v = 0; v < 4; ++v)
            if (v != o) mn = min(mn, g[v]);
        return mn;
    } else {
        return min(g[edge_start(KT::D, k)], g[edge_end(KT::D, k)]);
    }
}

// key of local entity k = its other (non-minimum) nodes, ascending
template <class KT>
__device__ __forceinline__ uint64_t entity_key(const int (&g)[KT::NV], int k) {
    if constexpr (KT::FACES) {
        const int o = 3 - k;
        int f[3], t = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v)
            if (v != o) f[t++] = g[v];
        const int lo = min(f[0], min(f[1], f[2])), hi = max(f[0], max(f[1], f[2]));
        const int mid = f[0] + f[1] + f[2] - lo - hi;
        return ((uint64_t)(uint32_t)mid << 32) | (uint32_t)hi;
    } else {
        return (uint64_t)(uint32_t)max(g[edge_start(KT::D, k)], g[edge_end(KT::D, k)]);
    }
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
        // base parity of (f0,f1,f2,opp): k=0 (0,1,2,3) even, k=1 (0,1,3,2) odd,
        // k=2 (0,2,3,1) even, k=3 (1,2,3,0) odd.
        const int o = 3 - k;
        int f[3], t = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v)
            if (v != o) f[t++] = g[v];
        const int inv = (f[0] > f[1]) + (f[0] > f[2]) + (f[1] > f[2]);
        return ((inv + (k & 1)) & 1) ? 1 : -1;  // s = -sgn(pi)
    } else {
        return g[edge_start(KT::D, k)] < g[edge_end(KT::D, k)] ? 1 : -1;
    }
}

// ---------------------------------------------------------------------------------
// counting sort of instances by minimum node (warp-aggregated atomics)
// ---------------------------------------------------------------------------------
template <class KT, bool FILL>
__global__ void __launch_bounds__(256) k_bucket(const int32_t* __restrict__ elems, int64_t n_elems, int64_t n_nodes,
                                                int32_t* __restrict__ cnt, const int32_t* __restrict__ bucket_ptr,
                                                int32_t* __restrict__ bucket, WsHeader* hdr) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool live = e < n_elems;
    int g[KT::NV];
    if (live) {
        load_elem<KT>(elems, (int)e, g);
        bool bad = false;
#pragma unroll
        for (int v = 0; v < KT::NV; ++v) bad |= (unsigned)g[v] >= (unsigned long long)n_nodes;
        if (bad) {
            atomicOr(&hdr->flags[F_INVALID_NODE], 1);
#pragma unroll
            for (int v = 0; v < KT::NV; ++v) g[v] = 0;
        }
    }
    if (!live) return;
#pragma unroll
    for (int k = 0; k < KT::M; ++k) {
        const int a = entity_min_node<KT>(g, k);
        if constexpr (!FILL) {
            atomicAdd(&cnt[a], 1);
        } else {
            const int pos = atomicAdd(&cnt[a], 1);
            bucket[__ldg(bucket_ptr + a) + pos] = (int)((e << 3) | k);
        }
    }
}

// ---------------------------------------------------------------------------------
// per node: sort bucket, number entities, incidence, row lengths, look-back
// ---------------------------------------------------------------------------------
template <class KT>
struct NodeCaps {
    // instances per node held in shared memory (one 64-bit sort key each;
    // faces add a 32-bit instance word); larger buckets take a global-memory
    // slow path
    static constexpr int CAP = KT::D == 2 ? 16 : (KT::FACES ? 32 : 48);
    static constexpr int TPB = KT::D == 2 ? 128 : 64;
};

struct NodeOut {
    int32_t* e2d;
    int32_t* inc_ptr;
    int32_t* row_ptr;
    int32_t* d2n;  // optional
    int2* rec;     // 2D edges / 3D faces: {first, last} instance of each row
    int* flags;    // WsHeader flags
    int32_t* bucket;
    int64_t* totals;  // [0] n_dofs, [1] nnz
    unsigned long long* status;
    int* ticket;
};

// Sort item of an instance.  Edges: one u64 (other node << 32 | e << 3 | k),
// so sorting the word sorts by (entity, element).  Faces: u64 (mid << 32 | hi)
// plus the instance word as tie-break.
// Bucket words are instances e << 3 | k; k_node_count sets bit 31 on the
// first instance of every entity run (consumers mask with INST_MASK).
constexpr int INST_MASK = 0x7fffffff;
constexpr unsigned RUN_FLAG = 0x80000000u;

template <class KT>
struct Item {
    uint64_t key;
    int inst;
    __device__ __forceinline__ bool operator<(const Item& o) const {
        if constexpr (KT::FACES) return key < o.key || (key == o.key && inst < o.inst);
        else return key < o.key;
    }
    __device__ __forceinline__ uint64_t entity() const {  // entity key only
        if constexpr (KT::FACES) return key;
        else return key >> 32;
    }
};

template <class KT>
__device__ __forceinline__ Item<KT> make_item(const int32_t* __restrict__ elems, int inst) {
    inst &= INST_MASK;
    int g[KT::NV];
    load_elem<KT>(elems, inst >> 3, g);
    Item<KT> it;
    if constexpr (KT::FACES) {
        it.key = entity_key<KT>(g, inst & 7);
        it.inst = inst;
    } else {
        it.key = (entity_key<KT>(g, inst & 7) << 32) | (uint32_t)inst;
        it.inst = inst;
    }
    return it;
}

// number of distinct link vertices (nodes other than a, b) over the tets of
// one edge run; every tet contributes exactly two
template <class KT, class InstAt>
__device__ __forceinline__ int link_count(const int32_t* __restrict__ elems, int a, int b, int j, int q,
                                          InstAt inst_at) {
    constexpr int CAPL = 2 * EFEM_MAX_ROW_ELEMS;
    int lk[CAPL];
    int nl = 0, L = 0;
    for (int u = j; u < q; ++u) {
        int h[4];
        load_elem<KT>(elems, inst_at(u) >> 3, h);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int c = h[v];
            if (c == a || c == b) continue;
            bool seen = false;
            for (int w = 0; w < nl; ++w) seen |= lk[w] == c;
            if (!seen) {
                ++L;
                if (nl < CAPL) lk[nl++] = c;
            }
        }
    }
    return L;
}

// t <= 8: the 2t link values in registers, distinct count by pairwise compares
template <class KT, class InstAt>
__device__ __forceinline__ int link_count_fast(const int32_t* __restrict__ elems, int a, int b, int j, int q,
                                               InstAt inst_at) {
    const int t = q - j;
    if (t > 8) return link_count<KT>(elems, a, b, j, q, inst_at);
    int lk[16];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        if (u < t) {
            int h[4];
            load_elem<KT>(elems, inst_at(j + u) >> 3, h);
            // the two vertices other than a and b, in local order
            int c = -1, d = -1;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const bool link = h[v] != a && h[v] != b;
                d = (link && c >= 0 && d < 0) ? h[v] : d;
                c = (link && c < 0) ? h[v] : c;
            }
            lk[2 * u] = c;
            lk[2 * u + 1] = d;
        } else {
            lk[2 * u] = -1 - 2 * u;  // distinct sentinels never counted
            lk[2 * u + 1] = -2 - 2 * u;
        }
    }
    int L = 0;
#pragma unroll
    for (int x = 0; x < 16; ++x) {
        bool dup = false;
#pragma unroll
        for (int y = 0; y < x; ++y) dup |= lk[y] == lk[x];
        L += (x < 2 * t) && !dup;
    }
    return L;
}

// Pass A: per node, sort its bucket in place by (entity, element) and count
// its entities and the CSR entries of their rows.
template <class KT>
__global__ void __launch_bounds__(NodeCaps<KT>::TPB) k_node_count(const int32_t* __restrict__ elems,
                                                                  const int32_t* __restrict__ bucket_ptr,
                                                                  int32_t* __restrict__ bucket, int64_t n_nodes,
                                                                  int32_t* __restrict__ ent_cnt,
                                                                  int32_t* __restrict__ nnz_cnt) {
    constexpr int CAP = NodeCaps<KT>::CAP;
    constexpr int TPB = NodeCaps<KT>::TPB;
    __shared__ uint64_t s_key[CAP * TPB];
    __shared__ int s_inst[KT::FACES ? CAP * TPB : 1];
    const int64_t a64 = (int64_t)blockIdx.x * TPB + threadIdx.x;
    if (a64 >= n_nodes) return;
    const int a = (int)a64;
    const int beg = __ldg(bucket_ptr + a);
    const int n = __ldg(bucket_ptr + a + 1) - beg;
    int32_t* gb = bucket + beg;
    int n_ent = 0, n_nnz = 0;
    constexpr int NREG = 8;
    if (KT::D == 2 && n <= NREG) {
        // register path: bitonic network over 8 keys
        uint64_t rk[NREG];
#pragma unroll
        for (int j = 0; j < NREG; ++j) rk[j] = j < n ? make_item<KT>(elems, __ldg(gb + j)).key : ~0ull;
#pragma unroll
        for (int kk = 2; kk <= NREG; kk <<= 1)
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1)
#pragma unroll
                for (int x = 0; x < NREG; ++x) {
                    const int y = x ^ jj;
                    if (y > x) {
                        const bool sw = rk[x] > rk[y];
                        const bool asc = (x & kk) == 0;
                        const uint64_t lo = sw ? rk[y] : rk[x], hi = sw ? rk[x] : rk[y];
                        rk[x] = asc ? lo : hi;
                        rk[y] = asc ? hi : lo;
                    }
                }
#pragma unroll
        for (int x = 0; x < NREG; ++x)
            if (x < n) {
                const bool st = x == 0 || (rk[x] >> 32) != (rk[x - 1] >> 32);
                n_ent += st;
                gb[x] = (int)((uint32_t)rk[x] | (st ? RUN_FLAG : 0u));
            }
        n_nnz = n_ent + (KT::M - 1) * n;
    } else {
        const bool in_smem = n <= CAP;
        uint64_t* K = s_key + threadIdx.x;  // item j at [j * TPB]
        int* V = s_inst + (KT::FACES ? threadIdx.x : 0);
        auto get = [&](int j) -> Item<KT> {
            if (in_smem) {
                Item<KT> it;
                it.key = K[j * TPB];
                if constexpr (KT::FACES) it.inst = V[j * TPB];
                else it.inst = (int)(uint32_t)it.key;
                return it;
            }
            return make_item<KT>(elems, gb[j]);
        };
        auto put = [&](int j, const Item<KT>& it) {
            if (in_smem) {
                K[j * TPB] = it.key;
                if constexpr (KT::FACES) V[j * TPB] = it.inst;
            } else {
                gb[j] = it.inst;
            }
        };
        if (in_smem) {
#pragma unroll 4
            for (int j = 0; j < n; ++j) {
                const Item<KT> it = make_item<KT>(elems, __ldg(gb + j));
                K[j * TPB] = it.key;
                if constexpr (KT::FACES) V[j * TPB] = it.inst;
            }
        }
        for (int j = in_smem ? 1 : 0; j < n; ++j) {
            const Item<KT> it = in_smem ? get(j) : make_item<KT>(elems, gb[j]);
            int q = j;
            while (q > 0) {
                const Item<KT> prev = get(q - 1);
                if (!(it < prev)) break;
                put(q, prev);
                --q;
            }
            put(q, it);
        }
        auto inst_at = [&](int j) -> int { return (in_smem ? get(j).inst : gb[j]) & INST_MASK; };
        for (int j = 0; j < n;) {
            const uint64_t ek = get(j).entity();
            int q = j + 1;
            while (q < n && get(q).entity() == ek) ++q;
            if constexpr (KT::D == 3 && !KT::FACES)
                n_nnz += 1 + 2 * link_count_fast<KT>(elems, a, (int)ek, j, q, inst_at) + (q - j);
            ++n_ent;
            if (in_smem)
                for (int u = j; u < q; ++u) gb[u] = (int)((uint32_t)get(u).inst | (u == j ? RUN_FLAG : 0u));
            else
                gb[j] = (int)((uint32_t)gb[j] | RUN_FLAG);
            j = q;
        }
        if constexpr (!(KT::D == 3 && !KT::FACES)) n_nnz = n_ent + (KT::M - 1) * n;
    }
    ent_cnt[a] = n_ent;
    if constexpr (KT::D == 3 && !KT::FACES) nnz_cnt[a] = n_nnz;
}

// Pass B: per node, walk its sorted bucket: DOF ids (ent_ptr[a] + run),
// elems2dofs, the incidence offsets, dofs2nodes (on request).  Runs are read
// from the RUN_FLAG bits pass A left, so no element is gathered except for
// NE0 3D row lengths (link vertices) and dofs2nodes.  Only NE0 3D writes
// row_ptr here; for 2D edges and 3D faces row i starts at
// i + (m-1) inc_ptr[i] (closed form, written by the numeric kernel).
template <class KT>
__global__ void __launch_bounds__(256) k_node_write(const int32_t* __restrict__ elems,
                                                    const int32_t* __restrict__ bucket_ptr,
                                                    const int32_t* __restrict__ bucket,
                                                    const int32_t* __restrict__ ent_ptr,
                                                    const int32_t* __restrict__ nnz_ptr, int64_t n_nodes,
                                                    NodeOut out) {
    constexpr bool NE3 = KT::D == 3 && !KT::FACES;
    const int64_t a64 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a64 >= n_nodes) return;
    const int a = (int)a64;
    const int beg = __ldg(bucket_ptr + a);
    const int n = __ldg(bucket_ptr + a + 1) - beg;
    const int32_t* gb = bucket + beg;
    int id = __ldg(ent_ptr + a) - 1;
    int nnz_run = NE3 ? __ldg(nnz_ptr + a) : 0;
    auto inst_at = [&](int j) -> int { return __ldg(gb + j) & INST_MASK; };
    int run0 = 0, run_b = 0, first = 0, prev = 0;
    for (int j = 0; j < n; ++j) {
        const int w = __ldg(gb + j);
        const int inst = w & INST_MASK;
        if (w < 0) {  // RUN_FLAG: first instance of a new entity
            if constexpr (NE3) {
                if (j > 0) nnz_run += 1 + 2 * link_count_fast<KT>(elems, a, run_b, run0, j, inst_at) + (j - run0);
            } else {
                if (j > 0) {
                    out.rec[id] = make_int2(first, prev);
                    // a conforming mesh has <= 2 elements per edge (2D) / face (3D)
                    if (j - run0 > 2) atomicOr(&out.flags[F_ROW_MISMATCH], 1);
                }
                first = inst;
            }
            ++id;
            run0 = j;
            out.inc_ptr[id] = beg + j;
            if (NE3 || out.d2n) {
                int g[KT::NV];
                load_elem<KT>(elems, inst >> 3, g);
                const uint64_t key = entity_key<KT>(g, inst & 7);
                run_b = (int)key;
                if (NE3) out.row_ptr[id] = nnz_run;
                if (out.d2n) {
                    int32_t* row = out.d2n + (int64_t)id * KT::EK;
                    row[0] = a;
                    if constexpr (KT::FACES) {
                        row[1] = (int)(key >> 32);
                        row[2] = (int)(key & 0xffffffffu);
                    } else {
                        row[1] = (int)key;
                    }
                }
            }
        }
        out.e2d[(int64_t)(inst >> 3) * KT::M + (inst & 7)] = id;
        prev = inst;
    }
    if constexpr (NE3) {
        if (n > 0) nnz_run += 1 + 2 * link_count_fast<KT>(elems, a, run_b, run0, n, inst_at) + (n - run0);
    } else {
        if (n > 0) {
            out.rec[id] = make_int2(first, prev);
            if (n - run0 > 2) atomicOr(&out.flags[F_ROW_MISMATCH], 1);
        }
    }
    if (a == n_nodes - 1) {
        const int R = id + 1;
        out.inc_ptr[R] = beg + n;
        if (NE3) out.row_ptr[R] = nnz_run;
        out.totals[0] = R;
        // 2D edges / 3D faces: nnz = sum_i (1 + (m-1) t_i) = R + (m-1) (T m)
        out.totals[1] = NE3 ? (int64_t)nnz_run : (int64_t)R + (int64_t)(KT::M - 1) * (beg + n);
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

// ---------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------
// header reset + zero the two counter arrays (bucket counts, fill cursors)
__global__ void k_init(WsHeader* hdr, int32_t* __restrict__ cnt, int32_t* __restrict__ cursor, int64_t n1) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < F_NFLAGS) hdr->flags[i] = 0;
    if (i == 0) {
        hdr->bad_element = ~0ull;
        hdr->totals[0] = 0;
        hdr->totals[1] = 0;
    }
    if (i < n1) {
        cnt[i] = 0;
        cursor[i] = 0;
    }
}

template <class KT>
efem_status run_enumerate_kt(Plan& p, cudaStream_t s) {
    const int64_t N = p.n_nodes, T = p.n_elems;
    size_t bytes = p.cub_bytes;
    k_init<<<grid_for(N + 1 > F_NFLAGS ? N + 1 : F_NFLAGS, 256), 256, 0, s>>>(p.hdr, p.cnt, p.nnz_cnt, N + 1);
    EFEM_LAUNCH_CHECK();
    if (T > 0) {
        k_bucket<KT, false><<<grid_for(T, 256), 256, 0, s>>>(p.elems, T, N, p.cnt, nullptr, nullptr, p.hdr);
        EFEM_LAUNCH_CHECK();
    }
    EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.cnt, p.bucket_ptr, (int)(N + 1), s));
    count_launch(2);
    if (T > 0) {  // fill cursors: nnz_cnt (zeroed by k_init, overwritten by pass A)
        k_bucket<KT, true><<<grid_for(T, 256), 256, 0, s>>>(p.elems, T, N, p.nnz_cnt, p.bucket_ptr, p.bucket,
                                                             p.hdr);
        EFEM_LAUNCH_CHECK();
    }
    if (N == 0) {
        EFEM_CUDA_TRY(cudaMemsetAsync(p.inc_ptr, 0, 4, s));
        EFEM_CUDA_TRY(cudaMemsetAsync(p.row_ptr, 0, 4, s));
        return EFEM_OK;
    }
    // pass A: sort buckets, count entities / row entries per node (cnt reused
    // for the entity counts; cnt[N] = nnz_cnt[N] = 0 from k_init)
    constexpr int TPB = NodeCaps<KT>::TPB;
    k_node_count<KT><<<grid_for(N, TPB), TPB, 0, s>>>(p.elems, p.bucket_ptr, p.bucket, N, p.cnt, p.nnz_cnt);
    EFEM_LAUNCH_CHECK();
    EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.cnt, p.ent_ptr, (int)(N + 1), s));
    count_launch(2);
    if constexpr (KT::D == 3 && !KT::FACES) {  // row lengths need a union only for 3D edges
        EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.nnz_cnt, p.nnz_ptr, (int)(N + 1), s));
        count_launch(2);
    }
    // pass B: DOF ids, elems2dofs, incidence (+ row_ptr for 3D edges)
    NodeOut o{p.e2d,    p.inc_ptr, p.row_ptr,  p.want_d2n ? p.d2n : nullptr, p.rec, reinterpret_cast<int*>(reinterpret_cast<char*>(p.hdr) + offsetof(WsHeader, flags)),
              p.bucket, p.d_totals, nullptr,    nullptr};
    k_node_write<KT><<<grid_for(N, 256), 256, 0, s>>>(p.elems, p.bucket_ptr, p.bucket, p.ent_ptr, p.nnz_ptr, N, o);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status launch_enumerate(Plan& p, cudaStream_t s) {
    if (p.dim == 2) return p.element == EFEM_RT0 ? run_enumerate_kt<Kind<2, EFEM_RT0>>(p, s)
                                                 : run_enumerate_kt<Kind<2, EFEM_NED0>>(p, s);
    return p.element == EFEM_RT0 ? run_enumerate_kt<Kind<3, EFEM_RT0>>(p, s)
                                 : run_enumerate_kt<Kind<3, EFEM_NED0>>(p, s);
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

}  // namespace efem
