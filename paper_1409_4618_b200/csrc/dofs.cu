// dofs.cu -- DOF enumeration, orientation and CSR row lengths
// (get_edges / get_faces / signs_edges /
// signs_faces of Sec. 3; PAPER.md:696 for the sparse pattern).
//
// Global DOF = edge (2D, 3D NE0) or face (3D RT0), numbered by the
// lexicographic rank of its ascending node tuple (reading C10).  Instead of a
// global radix sort of T*m keys, every (element,
// local entity) INSTANCE is bucketed by the entity's minimum node a with one
// counting sort, then sorted inside its bucket:
//   k_bucket<count>  instances per minimum node (one atomic per distinct
//                    minimum node of an element, not per instance)
//   CUB scan         -> bucket_ptr
//   k_bucket<fill>   scatter each instance's sort key (its other nodes, and
//                    e << 3 | k) into the buckets -- no later pass gathers
//                    elements again
//   k_node_count     per node: sort its bucket by (other nodes, element id);
//                    runs of equal keys are its entities, numbered
//                    ent_ptr[a] + run index, which IS the lexicographic rank.
//                    Writes the sorted instances (the entity -> element
//                    incidence, ascending element id per entity) with a
//                    RUN_FLAG on each run start.  Row lengths (no union):
//                      2D edges / 3D faces: 1 + (m-1) t   (two elements share
//                        at most one entity of that kind),
//                      3D edges: 1 + 2 L + t, L the distinct link vertices
//                        (each gives edges a-c, b-c; each tet adds its link
//                        edge).  The link of an edge is a cycle (interior:
//                        L = t) or a path (boundary: L = t + 1); the XOR of
//                        all link-vertex occurrences is 0 exactly for the
//                        cycle, so L = t + [xor != 0] (BND_FLAG).  The numeric
//                        kernel re-derives every row's column set and flags
//                        a mismatch (non-manifold fans) as non-conforming.
//   CUB scan(s) of the node tiles' totals (+ nnz totals for 3D edges);
//                       k_node_write finishes ent_ptr with a CTA scan
//   k_node_write     DOF ids, elems2dofs, inc_ptr, row records / row_ptr
#include <cub/cub.cuh>

#include "efem_internal.cuh"

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
// counting sort of instances by minimum node
// ---------------------------------------------------------------------------------
struct BucketArrays {
    uint64_t* key;  // edges: other node << 32 | inst; faces: mid << 32 | hi
    int32_t* inst;  // (unused: 3D records carry it)
    int32_t* x;     // 3D edges, exact mode: the runs' link excess
};
// 2D: one u64 key per instance.  3D: a 16-byte record {key, aux} per
// instance (aux = e << 3 | k for faces, the xor of the tet's four vertex ids
// for edges), so the scattered fill issues one store per instance.
template <class KT>
constexpr int KS = KT::D == 3 ? 2 : 1;  // key stride in u64 words

template <class KT, bool FILL>
__device__ __forceinline__ void bucket_one(const int32_t* __restrict__ elems, int64_t e, int64_t n_nodes,
                                           int32_t* __restrict__ cnt, const int32_t* __restrict__ bucket_ptr,
                                           BucketArrays B, WsHeader* hdr) {
    constexpr int M = KT::M;
    int g[KT::NV];
    load_elem<KT>(elems, (int)e, g);
    bool bad = false;
#pragma unroll
    for (int v = 0; v < KT::NV; ++v) bad |= (unsigned)g[v] >= (unsigned long long)n_nodes;
    if (bad) {
        if (!FILL) atomicOr(&hdr->flags[F_INVALID_NODE], 1);
#pragma unroll
        for (int v = 0; v < KT::NV; ++v) g[v] = 0;
    }
    int amin[M];
#pragma unroll
    for (int k = 0; k < M; ++k) amin[k] = entity_min_node<KT>(g, k);
    // one atomic per distinct minimum node of the element; its instances take
    // consecutive slots in local order
    int slot[M];
    bool owner[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
        bool first = true;
        int before = 0, total = 0;
#pragma unroll
        for (int q = 0; q < M; ++q) {
            const bool same = amin[q] == amin[k];
            if (q < k) {
                first &= !same;
                before += same;
            }
            total += same;
        }
        owner[k] = first;
        // count: add; fill: take slots from the top of the bucket (the counts
        // return to zero, which the next enumeration's count pass relies on)
        slot[k] = first ? (FILL ? atomicSub(&cnt[amin[k]], total) - total : atomicAdd(&cnt[amin[k]], total)) : before;
    }
    if constexpr (FILL) {
#pragma unroll
        for (int k = 0; k < M; ++k) {
            int base = slot[k];
            if (!owner[k]) {
#pragma unroll
                for (int q = 0; q < M; ++q)
                    if (q < k && owner[q] && amin[q] == amin[k]) base = slot[q] + slot[k];
            }
            const int64_t pos = (int64_t)__ldg(bucket_ptr + amin[k]) + base;
            const int inst = (int)((e << 3) | k);
            if constexpr (KT::FACES) {
                reinterpret_cast<ulonglong2*>(B.key)[pos] =
                    make_ulonglong2(entity_key<KT>(g, k), (unsigned long long)(uint32_t)inst);
            } else if constexpr (KT::D == 3) {
                reinterpret_cast<ulonglong2*>(B.key)[pos] =
                    make_ulonglong2((entity_key<KT>(g, k) << 32) | (uint32_t)inst,
                                    (unsigned long long)(uint32_t)(g[0] ^ g[1] ^ g[2] ^ g[3]));
            } else {
                B.key[pos] = (entity_key<KT>(g, k) << 32) | (uint32_t)inst;
            }
        }
    }
}

template <class KT, bool FILL>
__global__ void __launch_bounds__(256) k_bucket(const int32_t* __restrict__ elems, int64_t n_elems, int64_t n_nodes,
                                                int32_t* __restrict__ cnt, const int32_t* __restrict__ bucket_ptr,
                                                BucketArrays B, WsHeader* hdr) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    bucket_one<KT, FILL>(elems, e, n_nodes, cnt, bucket_ptr, B, hdr);
}

// ---------------------------------------------------------------------------------
// NE0 3D, one pass over the tets: the instance counts of the bucket layout
// (as k_bucket<count>) plus each tet's id in FIXED-capacity fans of its three
// smallest vertices (the nodes whose edges it holds): the node pass then
// gathers the tets instead of reading 16-byte instance records, and the
// record fill disappears.  A fan over C tets, or a tet with repeated (or
// out-of-range, counted as node 0) vertices, sets F_FAN_OVER: the record
// fill (k_bucket_cond) then runs on the device and the node pass reads the
// records, exactly the counting-sort path.
// ---------------------------------------------------------------------------------
constexpr int NE3_FAN_C = 24;  // fan slots per node (structured tet meshes: 18)

__global__ void __launch_bounds__(256) k_fill_fan3(const int32_t* __restrict__ elems, int64_t n_elems, int64_t n_nodes,
                                                   int32_t* __restrict__ cnt, int32_t* __restrict__ fcnt,
                                                   int32_t* __restrict__ fan, WsHeader* hdr) {
    using KT = Kind<3, EFEM_NED0>;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    bucket_one<KT, false>(elems, e, n_nodes, cnt, nullptr, BucketArrays{}, hdr);  // instance counts
    int g[4];
    load_elem<KT>(elems, (int)e, g);
    bool over = false;
#pragma unroll
    for (int v = 0; v < 4; ++v) over |= (unsigned)g[v] >= (unsigned long long)n_nodes;
    over |= g[0] == g[1] || g[0] == g[2] || g[0] == g[3] || g[1] == g[2] || g[1] == g[3] || g[2] == g[3];
    if (!over) {
        const int mx = max(max(g[0], g[1]), max(g[2], g[3]));
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            if (g[v] != mx) {  // one of the three smallest
                const int k = atomicAdd(fcnt + g[v], 1);
                if (k < NE3_FAN_C) fan[(int64_t)g[v] * NE3_FAN_C + k] = (int)e;
                else over = true;
            }
        }
    }
    if (over) atomicOr(&hdr->flags[F_FAN_OVER], 1);
}

// the record fill of the counting-sort path, only after an overflow
template <class KT>
__global__ void __launch_bounds__(256) k_bucket_cond(const int32_t* __restrict__ elems, int64_t n_elems,
                                                     int64_t n_nodes, int32_t* __restrict__ cnt,
                                                     const int32_t* __restrict__ bucket_ptr, BucketArrays B,
                                                     WsHeader* hdr) {
    if (!__ldg(&hdr->flags[F_FAN_OVER])) return;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_elems; e += (int64_t)gridDim.x * blockDim.x)
        bucket_one<KT, true>(elems, e, n_nodes, cnt, bucket_ptr, B, hdr);
}

// ---------------------------------------------------------------------------------
// per node: sort the bucket, count entities and row entries
// ---------------------------------------------------------------------------------
template <class KT>
struct NodeCaps {
    // instances per node held in shared memory; larger buckets take a
    // global-memory slow path
    static constexpr int CAP = KT::D == 2 ? 16 : (KT::FACES ? 32 : 48);
    static constexpr int TPB = KT::D == 2 ? 128 : 64;
    static constexpr int DCAP = 12;  // 3D edges: distinct larger neighbours held in registers
};

struct NodeOut {
    int32_t* e2d;
    int32_t* inc_ptr;
    int32_t* row_ptr;
    int32_t* d2n;  // optional
    int32_t* nbr;  // 3D edges: larger endpoint b of every edge (DOF id order)
    int2* rec;     // 2D edges / 3D faces: {first, last} instance of each row
    int* flags;    // WsHeader flags
    int32_t* bucket;
    int64_t* totals;  // [0] n_dofs, [1] nnz
};

// Bucket words after k_node_count: instances e << 3 | k (INST_MASK); bit 31
// marks the first instance of every entity run, bit 30 (3D edges, on run
// starts) a boundary edge (open link path).
constexpr unsigned RUN_FLAG = 0x80000000u;
constexpr unsigned BND_FLAG = 0x40000000u;

// Sort item of an instance.  Edges: one u64 (other node << 32 | e << 3 | k),
// so sorting the word sorts by (entity, element).  Faces: u64 (mid << 32 | hi)
// plus the instance word as tie-break.
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
__device__ __forceinline__ Item<KT> load_item(const BucketArrays& B, int64_t pos) {
    Item<KT> it;
    it.key = B.key[pos * KS<KT>];
    if constexpr (KT::FACES) it.inst = (int)(uint32_t)B.key[pos * KS<KT> + 1];
    else it.inst = (int)(uint32_t)it.key;
    return it;
}

// 2D edges, 3D faces: sort by (entity, element), flag runs.
template <class KT, bool SMEM>
__device__ __forceinline__ void node_sort_generic(const BucketArrays& B, int32_t* __restrict__ gb, int64_t beg,
                                                  int n, uint64_t* s_key, int* s_inst, int& n_ent) {
    constexpr int CAP = NodeCaps<KT>::CAP;
    constexpr int TPB = NodeCaps<KT>::TPB;
    const bool in_smem = SMEM && n <= CAP;
    uint64_t* K = s_key + threadIdx.x;  // item j at [j * TPB]
    int* V = s_inst + (KT::FACES ? threadIdx.x : 0);
    // slow path (n > CAP): sort in place in the bucket-key arrays (global)
    auto get = [&](int j) -> Item<KT> {
        if (in_smem) {
            Item<KT> it;
            it.key = K[j * TPB];
            if constexpr (KT::FACES) it.inst = V[j * TPB];
            else it.inst = (int)(uint32_t)it.key;
            return it;
        }
        return load_item<KT>(B, beg + j);
    };
    auto put = [&](int j, const Item<KT>& it) {
        if (in_smem) {
            K[j * TPB] = it.key;
            if constexpr (KT::FACES) V[j * TPB] = it.inst;
        } else {
            B.key[(beg + j) * KS<KT>] = it.key;
            if constexpr (KT::FACES) B.key[(beg + j) * KS<KT> + 1] = (uint32_t)it.inst;
        }
    };
    if (in_smem) {
#pragma unroll 4
        for (int j = 0; j < n; ++j) put(j, load_item<KT>(B, beg + j));
    }
    for (int j = 1; j < n; ++j) {
        const Item<KT> it = get(j);
        int q = j;
        while (q > 0) {
            const Item<KT> prev = get(q - 1);
            if (!(it < prev)) break;
            put(q, prev);
            --q;
        }
        put(q, it);
    }
    uint64_t prev = 0;
    for (int j = 0; j < n; ++j) {
        const Item<KT> it = get(j);
        const bool st = j == 0 || it.entity() != prev;
        prev = it.entity();
        n_ent += st;
        gb[j] = (int)((uint32_t)it.inst | (st ? RUN_FLAG : 0u));
    }
}

// 3D edges: group the node's instances by the other node b -- sorted
// distinct list D (<= DCAP) in shared memory, then a counting scatter.  The
// order inside a group (the tets of one edge) is left as the fill produced
// it; the numeric kernel sorts each row's tets by element id, so sums stay
// in a fixed order.  Also per group: t, and the xor of its link edges
// (BND_FLAG, see the file comment).  Writes the grouped instance words (RUN
// flag on group starts) and group q's b at x[q] (compact, so the write-back
// is a sector or two per node; read by k_node_write).  Returns false when the node has more than DCAP
// distinct larger neighbours (caller falls back to the generic sort).
template <class KT, int DC>
__device__ __forceinline__ bool node_group_ne3(const BucketArrays& B, int32_t* __restrict__ gb, int64_t beg, int n,
                                               int a, int* s_grp, int& n_ent, int& n_nnz) {
    // The distinct list D (ascending) and the per-group counts live in
    // registers (fully unrolled, compile-time indices): searches and
    // insertions are compare / select chains with no dependent shared-memory
    // round trips.  The scatter cursors and link xors use shared memory.
    constexpr int TPB = NodeCaps<KT>::TPB;
    static_assert(DC <= NodeCaps<KT>::DCAP, "shared scratch sized for DCAP groups");
    int* Cur = s_grp + threadIdx.x;                   // [p * TPB]: running cursor of group p
    int* X = Cur + NodeCaps<KT>::DCAP * TPB;          // xor of link edges of group p
    const ulonglong2* __restrict__ rec = reinterpret_cast<const ulonglong2*>(B.key) + beg;
    int D[DC], C[DC];
#pragma unroll
    for (int q = 0; q < DC; ++q) {
        D[q] = INT_MAX;
        C[q] = 0;
    }
    int nd = 0;
    bool over = false;
    constexpr int U = 8;  // keys loaded ahead of use
    for (int j0 = 0; j0 < n; j0 += U) {
        int bb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) bb[u] = j0 + u < n ? (int)(__ldg(&rec[j0 + u].x) >> 32) : -1;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int b = bb[u];
            if (b < 0) continue;
            int lt = 0;
            bool found = false;
#pragma unroll
            for (int q = 0; q < DC; ++q) {  // D[q] = INT_MAX beyond nd
                lt += D[q] < b;
                found |= D[q] == b;
            }
            if (found) {
#pragma unroll
                for (int q = 0; q < DC; ++q) C[q] += q == lt;
            } else if (nd == DC) {
                over = true;
            } else {
#pragma unroll
                for (int q = DC - 1; q > 0; --q) {
                    D[q] = q > lt ? D[q - 1] : (q == lt ? b : D[q]);
                    C[q] = q > lt ? C[q - 1] : (q == lt ? 1 : C[q]);
                }
                D[0] = lt == 0 ? b : D[0];
                C[0] = lt == 0 ? 1 : C[0];
                ++nd;
            }
        }
    }
    if (over) return false;
    int S[DC];
    int off = 0;
#pragma unroll
    for (int q = 0; q < DC; ++q) {
        S[q] = off;
        if (q < nd) {
            Cur[q * TPB] = off;
            X[q * TPB] = 0;
        }
        off += C[q];
    }
    for (int j0 = 0; j0 < n; j0 += U) {
        uint64_t kk[U];
        int xx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const ulonglong2 r = j0 + u < n ? __ldg(rec + j0 + u) : make_ulonglong2(0ull, 0ull);
            kk[u] = r.x;
            xx[u] = (int)(uint32_t)r.y;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (j0 + u >= n) continue;
            const int b = (int)(kk[u] >> 32);
            int g = 0, st = 0;
#pragma unroll
            for (int q = 0; q < DC; ++q) g += D[q] < b;  // b present: its group index
#pragma unroll
            for (int q = 0; q < DC; ++q) st = q == g ? S[q] : st;
            const int pos = Cur[g * TPB];
            Cur[g * TPB] = pos + 1;
            X[g * TPB] ^= xx[u] ^ a ^ b;  // c ^ d of this tet
            gb[pos] = (int)((uint32_t)kk[u] | (pos == st ? RUN_FLAG : 0u));
        }
    }
    int nnz = 0;
#pragma unroll
    for (int q = 0; q < DC; ++q) {
        if (q < nd) {
            const int st = S[q];
            const bool bnd = X[q * TPB] != 0;  // open link path: L = t + 1
            if (bnd) atomicOr(gb + st, (int)BND_FLAG);
            B.x[beg + q] = D[q];  // compact: group q's b (the x words are consumed)
            nnz += 1 + 3 * C[q] + 2 * (int)bnd;
        }
    }
    n_ent = nd;
    n_nnz = nnz;
    return true;
}

// local edge of the local vertex pair (p, q), p != q: nibble 4 p + q
constexpr unsigned long long NE3_LOCAL_EDGE = 0x452403153002100ull;

// 3D edges, fan mode: node_group_ne3 over the node's fan tets (gathered)
// instead of its instance records -- instance (a, b) for every vertex b > a
// of a fan tet, inst = e << 3 | local edge, link-edge xor c ^ d = the tet's
// xor ^ a ^ b.  Same outputs (grouped words, BND / RUN flags, b's in x).
template <class KT, int DC>
__device__ __forceinline__ bool node_group_ne3_fan(const int32_t* __restrict__ elems, const int32_t* __restrict__ fl,
                                                   int nf, int32_t* __restrict__ gb, int32_t* __restrict__ bx, int a,
                                                   int* s_grp, int& n_ent, int& n_nnz) {
    constexpr int TPB = NodeCaps<KT>::TPB;
    static_assert(DC <= NodeCaps<KT>::DCAP, "shared scratch sized for DCAP groups");
    int* Cur = s_grp + threadIdx.x;
    int* X = Cur + NodeCaps<KT>::DCAP * TPB;
    int D[DC], C[DC];
#pragma unroll
    for (int q = 0; q < DC; ++q) {
        D[q] = INT_MAX;
        C[q] = 0;
    }
    int nd = 0;
    bool over = false;
    // tets gathered ahead of use (2: U = 1 / 4 / 8 measured 9 % / 14 % / 27 %
    // slower on the config-4 symbolic phase -- fewer unrolled compare chains
    // in flight beat deeper prefetch here)
    constexpr int U = 2;
    for (int f0 = 0; f0 < nf; f0 += U) {
        int4 tq[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            tq[u] = f0 + u < nf ? __ldg(reinterpret_cast<const int4*>(elems) + __ldg(fl + f0 + u))
                                : make_int4(-1, -1, -1, -1);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int gv[4] = {tq[u].x, tq[u].y, tq[u].z, tq[u].w};
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int b = gv[v];
                if (b <= a) continue;
                int lt = 0;
                bool found = false;
#pragma unroll
                for (int q = 0; q < DC; ++q) {
                    lt += D[q] < b;
                    found |= D[q] == b;
                }
                if (found) {
#pragma unroll
                    for (int q = 0; q < DC; ++q) C[q] += q == lt;
                } else if (nd == DC) {
                    over = true;
                } else {
#pragma unroll
                    for (int q = DC - 1; q > 0; --q) {
                        D[q] = q > lt ? D[q - 1] : (q == lt ? b : D[q]);
                        C[q] = q > lt ? C[q - 1] : (q == lt ? 1 : C[q]);
                    }
                    D[0] = lt == 0 ? b : D[0];
                    C[0] = lt == 0 ? 1 : C[0];
                    ++nd;
                }
            }
        }
    }
    if (over) return false;
    int S[DC];
    int off = 0;
#pragma unroll
    for (int q = 0; q < DC; ++q) {
        S[q] = off;
        if (q < nd) {
            Cur[q * TPB] = off;
            X[q * TPB] = 0;
        }
        off += C[q];
    }
    for (int f0 = 0; f0 < nf; f0 += U) {
        int ev[U];
        int4 tq[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ev[u] = f0 + u < nf ? __ldg(fl + f0 + u) : 0;
            tq[u] = f0 + u < nf ? __ldg(reinterpret_cast<const int4*>(elems) + ev[u]) : make_int4(-1, -1, -1, -1);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int gv[4] = {tq[u].x, tq[u].y, tq[u].z, tq[u].w};
            const int la = gv[0] == a ? 0 : (gv[1] == a ? 1 : (gv[2] == a ? 2 : 3));
            const int xr = gv[0] ^ gv[1] ^ gv[2] ^ gv[3];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int b = gv[v];
                if (b <= a) continue;
                int g = 0, st = 0;
#pragma unroll
                for (int q = 0; q < DC; ++q) g += D[q] < b;  // b present: its group index
#pragma unroll
                for (int q = 0; q < DC; ++q) st = q == g ? S[q] : st;
                const int pos = Cur[g * TPB];
                Cur[g * TPB] = pos + 1;
                X[g * TPB] ^= xr ^ a ^ b;  // c ^ d of this tet
                const int k = (int)((NE3_LOCAL_EDGE >> (4 * (la * 4 + v))) & 15ull);
                gb[pos] = (int)((uint32_t)((ev[u] << 3) | k) | (pos == st ? RUN_FLAG : 0u));
            }
        }
    }
    int nnz = 0;
#pragma unroll
    for (int q = 0; q < DC; ++q) {
        if (q < nd) {
            const int st = S[q];
            const bool bnd = X[q * TPB] != 0;  // open link path: L = t + 1
            if (bnd) atomicOr(gb + st, (int)BND_FLAG);
            bx[q] = D[q];  // compact: group q's b
            nnz += 1 + 3 * C[q] + 2 * (int)bnd;
        }
    }
    n_ent = nd;
    n_nnz = nnz;
    return true;
}

// fan mode, a node the register path cannot take (more distinct neighbours
// than DCAP, or exact link counts): its instance records {b << 32 | inst,
// tet xor} written into its bucket range of the key array, for the generic
// sort that follows
__device__ __forceinline__ void ne3_fan_records(const int32_t* __restrict__ elems, const int32_t* __restrict__ fl,
                                                int nf, int a, uint64_t* __restrict__ key, int64_t beg) {
    int j = 0;
    for (int f = 0; f < nf; ++f) {
        const int e = __ldg(fl + f);
        const int4 t = __ldg(reinterpret_cast<const int4*>(elems) + e);
        const int gv[4] = {t.x, t.y, t.z, t.w};
        const int la = gv[0] == a ? 0 : (gv[1] == a ? 1 : (gv[2] == a ? 2 : 3));
        const int xr = gv[0] ^ gv[1] ^ gv[2] ^ gv[3];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            if (gv[v] <= a) continue;
            const int k = (int)((NE3_LOCAL_EDGE >> (4 * (la * 4 + v))) & 15ull);
            key[(beg + j) * 2] = ((uint64_t)(uint32_t)gv[v] << 32) | (uint32_t)((e << 3) | k);
            key[(beg + j) * 2 + 1] = (uint64_t)(uint32_t)xr;
            ++j;
        }
    }
}

// 3D faces: group the node's instances by face key (mid << 32 | hi) with the
// sorted distinct list and counts in registers (as node_group_ne3), counting
// scatter, then each face's two tets in element order.  Returns false when
// the node has more than FDC distinct faces (caller sorts generically).
template <class KT, int FDC>
__device__ __forceinline__ bool node_group_faces(const BucketArrays& B, int32_t* __restrict__ gb, int64_t beg,
                                                 int n, int* s_cur, int& n_ent) {
    constexpr int TPB = NodeCaps<KT>::TPB;
    int* Cur = s_cur + threadIdx.x;  // [p * TPB]
    const ulonglong2* __restrict__ rec = reinterpret_cast<const ulonglong2*>(B.key) + beg;
    uint64_t D[FDC];
    int C[FDC];
#pragma unroll
    for (int q = 0; q < FDC; ++q) {
        D[q] = ~0ull;
        C[q] = 0;
    }
    int nd = 0;
    bool over = false;
    constexpr int U = 4;
    for (int j0 = 0; j0 < n; j0 += U) {
        uint64_t kk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) kk[u] = j0 + u < n ? __ldg(&rec[j0 + u].x) : ~0ull;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (j0 + u >= n) continue;
            const uint64_t b = kk[u];
            int lt = 0;
            bool found = false;
#pragma unroll
            for (int q = 0; q < FDC; ++q) {
                lt += D[q] < b;
                found |= D[q] == b;
            }
            if (found) {
#pragma unroll
                for (int q = 0; q < FDC; ++q) C[q] += q == lt;
            } else if (nd == FDC) {
                over = true;
            } else {
#pragma unroll
                for (int q = FDC - 1; q > 0; --q) {
                    D[q] = q > lt ? D[q - 1] : (q == lt ? b : D[q]);
                    C[q] = q > lt ? C[q - 1] : (q == lt ? 1 : C[q]);
                }
                D[0] = lt == 0 ? b : D[0];
                C[0] = lt == 0 ? 1 : C[0];
                ++nd;
            }
        }
    }
    if (over) return false;
    int S[FDC];
    int off = 0;
#pragma unroll
    for (int q = 0; q < FDC; ++q) {
        S[q] = off;
        if (q < nd) Cur[q * TPB] = off;
        off += C[q];
    }
    for (int j0 = 0; j0 < n; j0 += U) {
        uint64_t kk[U];
        int ii[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const ulonglong2 r = j0 + u < n ? __ldg(rec + j0 + u) : make_ulonglong2(0ull, 0ull);
            kk[u] = r.x;
            ii[u] = (int)(uint32_t)r.y;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (j0 + u >= n) continue;
            int g = 0;
#pragma unroll
            for (int q = 0; q < FDC; ++q) g += D[q] < kk[u];
            const int pos = Cur[g * TPB];
            Cur[g * TPB] = pos + 1;
            gb[pos] = ii[u];
        }
    }
    // order each face's elements (<= 2 in a conforming mesh; a longer run is
    // flagged by the write pass) and flag the run starts
#pragma unroll
    for (int q = 0; q < FDC; ++q) {
        if (q < nd) {
            const int st = S[q];
            if (C[q] == 2) {
                const int x = gb[st], y = gb[st + 1];
                gb[st] = (int)((uint32_t)min(x, y) | RUN_FLAG);
                gb[st + 1] = max(x, y);
            } else {  // t == 1, or t > 2 (non-conforming: flagged by the write pass)
                gb[st] = (int)((uint32_t)gb[st] | RUN_FLAG);
            }
        }
    }
    n_ent = nd;
    return true;
}

// 3D edges, fallback: after node_sort_generic, per run count the distinct
// link vertices exactly and set BND_FLAG = (L > t)
template <class KT>
__device__ __forceinline__ void ne3_runs_exact(const int32_t* __restrict__ elems, int32_t* __restrict__ gb, int n,
                                               int a, int32_t* __restrict__ xs, int& n_nnz) {
    int j = 0;
    while (j < n) {
        int q = j + 1;
        while (q < n && !(gb[q] < 0)) ++q;
        // edge (a, b): b from the first tet of the run
        const int i0 = gb[j] & INST_MASK;
        int g[4];
        load_elem<KT>(elems, i0 >> 3, g);
        const int b = (int)entity_key<KT>(g, i0 & 7);
        int L = 0;
        for (int u = j; u < q; ++u) {
            int h[4];
            load_elem<KT>(elems, (gb[u] & INST_MASK) >> 3, h);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int c = h[v];
                if (c == a || c == b) continue;
                bool seen = false;  // seen in an earlier tet of the run (or earlier in this one)
                for (int w = j; w < u && !seen; ++w) {
                    int f[4];
                    load_elem<KT>(elems, (gb[w] & INST_MASK) >> 3, f);
                    seen = f[0] == c || f[1] == c || f[2] == c || f[3] == c;
                }
                L += !seen;
            }
        }
        // the exact excess L - t (0 interior, 1 boundary, more at a
        // non-manifold edge) goes to the run start's x slot for pass B
        const int t = q - j;
        const int ex = L - t;
        if (ex > 0) gb[j] = (int)((uint32_t)gb[j] | BND_FLAG);
        xs[j] = ex;
        n_nnz += 1 + 2 * L + t;
        j = q;
    }
}

template <class KT>
__global__ void __launch_bounds__(NodeCaps<KT>::TPB) k_node_count(const int32_t* __restrict__ elems,
                                                                  const int32_t* __restrict__ bucket_ptr,
                                                                  BucketArrays B, int32_t* __restrict__ bucket,
                                                                  int64_t n_nodes, int32_t* __restrict__ ent_cnt,
                                                                  int32_t* __restrict__ nnz_cnt, int exact,
                                                                  int32_t* __restrict__ ent_bsum,
                                                                  int32_t* __restrict__ nnz_bsum,
                                                                  const int32_t* __restrict__ fan,
                                                                  const int32_t* __restrict__ fcnt, WsHeader* hdr) {
    constexpr bool NE3 = KT::D == 3 && !KT::FACES;
    constexpr int TPB = NodeCaps<KT>::TPB;
    constexpr int DCAP = NodeCaps<KT>::DCAP;
    using BlockReduce = cub::BlockReduce<int, TPB>;
    __shared__ typename BlockReduce::TempStorage red_tmp;
    __shared__ uint64_t s_key[1];  // (the generic fallback sorts in global memory)
    __shared__ int s_inst[1];
    __shared__ int s_grp[NE3 ? 2 * DCAP * TPB : 1];
    __shared__ int s_cur[KT::FACES ? 16 * TPB : 1];
    // NE3 fan mode (fan != NULL and no overflow): the node's tets come from
    // its fixed-capacity fan (k_fill_fan3), not from instance records.  (The
    // flag is read once per CTA.)
    __shared__ int s_fan;
    if (NE3 && threadIdx.x == 0) s_fan = fan && !*(volatile const int*)&hdr->flags[F_FAN_OVER];
    __syncthreads();
    const bool fanmode = NE3 && s_fan;
    const int64_t a64 = (int64_t)blockIdx.x * TPB + threadIdx.x;
    int n_ent = 0, n_nnz = 0;
    if (a64 < n_nodes) {
    const int a = (int)a64;
    const int64_t beg = __ldg(bucket_ptr + a);
    const int n = __ldg(bucket_ptr + a + 1) - (int)beg;
    int32_t* gb = bucket + beg;
    constexpr int NREG = 8;
    if constexpr (KT::D == 2) {
        if (n <= NREG) {
            // register path: bitonic network over 8 keys
            uint64_t rk[NREG];
#pragma unroll
            for (int j = 0; j < NREG; ++j) rk[j] = j < n ? B.key[beg + j] : ~0ull;
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
        } else {  // (rare: > 8 instances at a node) sort in global memory
            node_sort_generic<KT, false>(B, gb, beg, n, s_key, s_inst, n_ent);
        }
    } else if constexpr (KT::FACES) {
        // (fallback sorts in global memory: the fast path needs no key staging,
        // so the CTA keeps its shared memory small)
        // (12 distinct faces cover structured tet meshes; 16, then a generic sort)
        if (!node_group_faces<KT, 12>(B, gb, beg, n, s_cur, n_ent) &&
            !node_group_faces<KT, 16>(B, gb, beg, n, s_cur, n_ent))
            node_sort_generic<KT, false>(B, gb, beg, n, s_key, s_inst, n_ent);
    } else {
        // (8 distinct larger neighbours cover structured tet meshes; 12, then a generic sort)
        bool done;
        if (fanmode) {
            const int32_t* fl = fan + (int64_t)a * NE3_FAN_C;
            const int nf = __ldg(fcnt + a);
            done = !exact && (node_group_ne3_fan<KT, 8>(elems, fl, nf, gb, B.x + beg, a, s_grp, n_ent, n_nnz) ||
                              node_group_ne3_fan<KT, NodeCaps<KT>::DCAP>(elems, fl, nf, gb, B.x + beg, a, s_grp,
                                                                         n_ent, n_nnz));
            if (!done) ne3_fan_records(elems, fl, nf, a, B.key, beg);  // for the generic sort below
        } else {
            done = !exact && (node_group_ne3<KT, 8>(B, gb, beg, n, a, s_grp, n_ent, n_nnz) ||
                              node_group_ne3<KT, NodeCaps<KT>::DCAP>(B, gb, beg, n, a, s_grp, n_ent, n_nnz));
        }
        if (!done) {
            n_ent = 0;
            n_nnz = 0;
            // (the NE3 instantiation has no key smem: sort in global memory)
            node_sort_generic<KT, false>(B, gb, beg, n, s_key, s_inst, n_ent);
            ne3_runs_exact<KT>(elems, gb, n, a, B.x + beg, n_nnz);
            // the groups' b, compacted to the front of the range (as the fast
            // path leaves them; r <= j, so in place): in x, unless exact mode
            // keeps its excess counts there (then in the key records)
            for (int j = 0, r = 0; j < n; ++j)
                if (gb[j] < 0) {
                    const uint64_t kb = B.key[(beg + j) * 2];
                    if (exact) B.key[(beg + r++) * 2] = kb;
                    else B.x[beg + r++] = (int)(kb >> 32);
                }
        }
    }
    ent_cnt[a] = n_ent;
    if constexpr (NE3) nnz_cnt[a] = n_nnz;
    }
    // per-tile totals: the offsets come from a scan of these (one value per
    // CTA, not per node), finished inside the write pass
    const int et = BlockReduce(red_tmp).Sum(n_ent);
    if constexpr (NE3) {
        __syncthreads();
        const int nt = BlockReduce(red_tmp).Sum(n_nnz);
        if (threadIdx.x == 0) nnz_bsum[blockIdx.x] = nt;
    }
    if (threadIdx.x == 0) {
        ent_bsum[blockIdx.x] = et;
        if (blockIdx.x == 0) {  // the scans' trailing zero
            ent_bsum[gridDim.x] = 0;
            if (NE3) nnz_bsum[gridDim.x] = 0;
        }
    }
}

// Pass B: per node, walk its sorted bucket: DOF ids (ent_ptr[a] + run),
// elems2dofs, the incidence offsets, dofs2nodes (on request).  Runs and row
// lengths come from the flags pass A left, so no element is gathered except
// for dofs2nodes.  2D edges / 3D faces write row records {first, last}
// instance (row i starts at i + (m-1) inc_ptr[i], closed form); 3D edges
// write row_ptr.
template <class KT>
__global__ void __launch_bounds__(NodeCaps<KT>::TPB) k_node_write(const int32_t* __restrict__ elems,
                                                                  const int32_t* __restrict__ bucket_ptr,
                                                                  const int32_t* __restrict__ bucket,
                                                                  const uint64_t* __restrict__ bkey,
                                                                  const int32_t* __restrict__ bx,
                                                                  const int32_t* __restrict__ bnb,
                                                                  const int32_t* __restrict__ ent_cnt,
                                                                  const int32_t* __restrict__ nnz_cnt,
                                                                  const int32_t* __restrict__ ent_bpre,
                                                                  const int32_t* __restrict__ nnz_bpre,
                                                                  int32_t* __restrict__ ent_ptr, int64_t n_nodes,
                                                                  NodeOut out) {
    constexpr bool NE3 = KT::D == 3 && !KT::FACES;
    constexpr int TPB = NodeCaps<KT>::TPB;  // the same node tiles as k_node_count
    using BlockScan = cub::BlockScan<int, TPB>;
    __shared__ typename BlockScan::TempStorage scan_tmp;
    const int64_t a64 = (int64_t)blockIdx.x * TPB + threadIdx.x;
    const bool live = a64 < n_nodes;
    const int a = (int)a64;
    // node offsets: tile prefix (scanned tile totals) + scan within the tile
    int e_off, z_off = 0, e_tot;
    const int e_base = __ldg(ent_bpre + blockIdx.x);
    BlockScan(scan_tmp).ExclusiveSum(live ? __ldg(ent_cnt + a) : 0, e_off, e_tot);
    e_off += e_base;
    if constexpr (NE3) {
        __syncthreads();
        BlockScan(scan_tmp).ExclusiveSum(live ? __ldg(nnz_cnt + a) : 0, z_off);
        z_off += __ldg(nnz_bpre + blockIdx.x);
    }
    // The CTA's entities are the contiguous ids [e_base, e_base + e_tot); the
    // per-entity outputs (2D edges / 3D faces: row records and incidence
    // offsets; 3D edges: incidence offsets, row offsets, larger endpoints),
    // which consecutive threads would interleave, are staged in shared memory
    // and stored coalesced when they fit (capacity: the entities per node of
    // structured meshes times the CTA size)
    constexpr int SREC = NE3 ? 8 * TPB : (KT::FACES ? 16 * TPB : 4 * TPB);
    __shared__ int2 s_rec[SREC];  // 2D / faces: {first, last}; 3D edges: {row offset, larger endpoint}
    __shared__ int s_inc[SREC];
    const bool stage = e_tot <= SREC;
    if (live) {
    ent_ptr[a] = e_off;
    const int beg = __ldg(bucket_ptr + a);
    const int n = __ldg(bucket_ptr + a + 1) - beg;
    const int32_t* gb = bucket + beg;
    int id = e_off - 1;
    int nnz_run = z_off;
    int run0 = 0, first = 0, prev = 0, excess = 0, grp = 0;
    auto close_run = [&](int j_end) {
        const int t = j_end - run0;
        if constexpr (NE3) {
            nnz_run += 1 + 3 * t + 2 * excess;  // 1 + 2L + t, L = t + excess
        } else {
            if (stage) s_rec[id - e_base] = make_int2(first, prev);
            else out.rec[id] = make_int2(first, prev);
            // a conforming mesh has <= 2 elements per edge (2D) / face (3D)
            if (t > 2) atomicOr(&out.flags[F_ROW_MISMATCH], 1);
        }
    };
    auto visit = [&](int j, int w) {
        const int inst = w & INST_MASK;
        if (w < 0) {  // RUN_FLAG: first instance of a new entity
            if (j > 0) close_run(j);
            ++id;
            run0 = j;
            first = inst;
            if (stage) s_inc[id - e_base] = beg + j;
            else out.inc_ptr[id] = beg + j;
            if constexpr (NE3) {
                if (!stage) out.row_ptr[id] = nnz_run;
                // link excess L - t: the BND flag (0 / 1) on the manifold
                // closed form, the exact count in exact mode
                excess = bx ? __ldg(bx + beg + j) : (w & BND_FLAG ? 1 : 0);
                // b, compacted by pass A
                const int b = bx ? (int)(__ldg(bkey + (beg + grp) * 2) >> 32) : __ldg(bnb + beg + grp);
                ++grp;
                if (stage) s_rec[id - e_base] = make_int2(nnz_run, b);
                else out.nbr[id] = b;
                if (out.d2n) {
                    out.d2n[(int64_t)id * 2] = a;
                    out.d2n[(int64_t)id * 2 + 1] = b;
                }
            } else if (out.d2n) {
                int g[KT::NV];
                load_elem<KT>(elems, inst >> 3, g);
                const uint64_t key = entity_key<KT>(g, inst & 7);
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
        if constexpr (!NE3) out.e2d[(int64_t)(inst >> 3) * KT::M + (inst & 7)] = id;  // 3D edges: k_elem_dofs
        prev = inst;
    };
    // the words in chunks of 8, loaded ahead of their (dependent) processing
    constexpr int U = 8;
    for (int j0 = 0; j0 < n; j0 += U) {
        int wv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) wv[u] = j0 + u < n ? __ldg(gb + j0 + u) : 0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (j0 + u < n) visit(j0 + u, wv[u]);
    }
    if (n > 0) close_run(n);
    if (a == n_nodes - 1) {
        const int R = id + 1;
        ent_ptr[n_nodes] = R;
        out.inc_ptr[R] = beg + n;
        if (NE3) out.row_ptr[R] = nnz_run;
        out.totals[0] = R;
        // 2D edges / 3D faces: nnz = sum_i (1 + (m-1) t_i) = R + (m-1) (T m)
        out.totals[1] = NE3 ? (int64_t)nnz_run : (int64_t)R + (int64_t)(KT::M - 1) * (beg + n);
    }
    }
    if (stage) {
        __syncthreads();
        for (int x = threadIdx.x; x < e_tot; x += TPB) {
            const int2 r = s_rec[x];
            if constexpr (NE3) {
                out.row_ptr[e_base + x] = r.x;
                out.nbr[e_base + x] = r.y;
            } else {
                out.rec[e_base + x] = r;
            }
            out.inc_ptr[e_base + x] = s_inc[x];
        }
    }
}

// 3D edges: elems2dofs per element (coalesced writes): the DOF of edge (a, b)
// is ent_ptr[a] + the rank of b among a's larger neighbours nbr[ent_ptr[a] ..
// ent_ptr[a+1]) (ascending: they are the lexicographic ranks).
template <class KT>
__global__ void __launch_bounds__(256) k_elem_dofs(const int32_t* __restrict__ elems, int64_t n_elems,
                                                   const int32_t* __restrict__ ent_ptr,
                                                   const int32_t* __restrict__ nbr, int32_t* __restrict__ e2d,
                                                   const WsHeader* hdr) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    if (*(volatile const int*)&hdr->flags[F_INVALID_NODE]) return;  // raw ids index ent_ptr below
    int g[4];
    load_elem<KT>(elems, (int)e, g);
    int id[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const int u = g[edge_start(3, k)], v = g[edge_end(3, k)];
        const int a = min(u, v), b = max(u, v);
        int lo = __ldg(ent_ptr + a), hi = __ldg(ent_ptr + a + 1) - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(nbr + mid) < b) lo = mid + 1; else hi = mid;
        }
        id[k] = lo;
    }
    int2* o = reinterpret_cast<int2*>(e2d + e * 6);  // 8-byte aligned: 6 ints per element
    o[0] = make_int2(id[0], id[1]);
    o[1] = make_int2(id[2], id[3]);
    o[2] = make_int2(id[4], id[5]);
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
// header reset.  The instance counters need no reset: they are zeroed with
// the workspace and every enumeration's fill pass takes them back to zero.
__global__ void k_init(WsHeader* hdr) {
    const int i = threadIdx.x;
    if (i < F_NFLAGS) hdr->flags[i] = 0;
    if (i == 0) {
        hdr->bad_element = ~0ull;
        hdr->totals[0] = 0;
        hdr->totals[1] = 0;
    }
}

template <class KT>
efem_status run_enumerate_kt(Plan& p, cudaStream_t s) {
    const int64_t N = p.n_nodes, T = p.n_elems;
    size_t bytes = p.cub_bytes;
    const BucketArrays barr{p.bkey, p.binst, p.bx};
    k_init<<<1, 32, 0, s>>>(p.hdr);
    EFEM_LAUNCH_CHECK();
#ifndef EFEM_NE3_FAN
#define EFEM_NE3_FAN 1
#endif
    // NE0 3D: one-pass fan fill (k_fill_fan3); exact link counts keep the
    // record path
    constexpr bool NE3 = KT::D == 3 && !KT::FACES;
    const bool fan3 = NE3 && EFEM_NE3_FAN && !p.exact_ne3 && N > 0;
    // (2D plans: the node-fan pipeline's one-pass fill leaves its counts in
    // cnt; 3D plans keep the invariant that every fill returns them to zero)
    // (the 2D fan pipeline's one-pass fill and the NE3 fan fill leave their
    // counts in cnt -- and an NE3 plan switches between that and the record
    // path with efem_plan_set_exact; the counting-sort fills return them to zero)
    if (KT::D == 2 || NE3) EFEM_CUDA_TRY(cudaMemsetAsync(p.cnt, 0, (size_t)(N + 1) * 4, s));
    if (fan3) EFEM_CUDA_TRY(cudaMemsetAsync(p.ne3_fcnt, 0, (size_t)N * 4, s));
    if (T > 0) {
        if (fan3)
            k_fill_fan3<<<grid_for(T, 256), 256, 0, s>>>(p.elems, T, N, p.cnt, p.ne3_fcnt, p.ne3_fan, p.hdr);
        else
            k_bucket<KT, false><<<grid_for(T, 256), 256, 0, s>>>(p.elems, T, N, p.cnt, nullptr, BucketArrays{}, p.hdr);
        EFEM_LAUNCH_CHECK();
    }
    EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.cnt, p.bucket_ptr, (int)(N + 1), s));
    count_launch(2);
    if (T > 0) {
        if (fan3) {  // the record fill only after an overflow (exits at once otherwise)
            int sms = 148, dev = 0;
            if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            k_bucket_cond<KT><<<8 * sms, 256, 0, s>>>(p.elems, T, N, p.cnt, p.bucket_ptr, barr, p.hdr);
        } else {
            k_bucket<KT, true><<<grid_for(T, 256), 256, 0, s>>>(p.elems, T, N, p.cnt, p.bucket_ptr, barr, p.hdr);
        }
        EFEM_LAUNCH_CHECK();
    }
    if (N == 0) {
        EFEM_CUDA_TRY(cudaMemsetAsync(p.inc_ptr, 0, 4, s));
        EFEM_CUDA_TRY(cudaMemsetAsync(p.row_ptr, 0, 4, s));
        return EFEM_OK;
    }
    // pass A: sort buckets, count entities / row entries per node (cnt reused
    // entity counts in ent_cnt; ent_cnt[N] = nnz_cnt[N] = 0 since the workspace was set)
    constexpr int TPB = NodeCaps<KT>::TPB;
    const int nb = (int)grid_for(N, TPB);
    k_node_count<KT><<<nb, TPB, 0, s>>>(p.elems, p.bucket_ptr, barr, p.bucket, N, p.ent_cnt, p.nnz_cnt,
                                         (int)p.exact_ne3, p.ent_bsum, p.nnz_bsum, fan3 ? p.ne3_fan : nullptr,
                                         p.ne3_fcnt, p.hdr);
    EFEM_LAUNCH_CHECK();
    // scans over the CTA tiles' totals only (the write pass finishes per node)
    EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.ent_bsum, p.ent_bpre, nb + 1, s));
    count_launch(2);
    if constexpr (KT::D == 3 && !KT::FACES) {  // row lengths need a union only for 3D edges
        EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.nnz_bsum, p.nnz_bpre, nb + 1, s));
        count_launch(2);
    }
    // pass B: DOF ids, elems2dofs, incidence (+ row_ptr for 3D edges)
    int* d_flags = reinterpret_cast<int*>(reinterpret_cast<char*>(p.hdr) + offsetof(WsHeader, flags));
    NodeOut o{p.e2d, p.inc_ptr, p.row_ptr, p.want_d2n ? p.d2n : nullptr, p.nbr, p.rec, d_flags, p.bucket,
              p.d_totals};
    k_node_write<KT><<<nb, TPB, 0, s>>>(p.elems, p.bucket_ptr, p.bucket, p.bkey, p.exact_ne3 ? p.bx : nullptr, p.bx,
                                         p.ent_cnt, p.nnz_cnt, p.ent_bpre, p.nnz_bpre, p.ent_ptr, N, o);
    EFEM_LAUNCH_CHECK();
    if constexpr (KT::D == 3 && !KT::FACES) {
        if (T > 0) {
            k_elem_dofs<KT><<<grid_for(T, 256), 256, 0, s>>>(p.elems, T, p.ent_ptr, p.nbr, p.e2d, p.hdr);
            EFEM_LAUNCH_CHECK();
        }
    }
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
