// fan2d.cu -- the symbolic half of the 2D hot path (RT0 and NE0 on
// triangles) as a node-fan pipeline: DOF enumeration and the sparsity
// pattern's row structure in two kernels (plus an on-device fallback).
//
// The method (Sec. 2.4; 671-696, Sec. 3.2): global edge
// DOFs numbered by the lexicographic rank of their sorted node pair (reading
// C10), local matrices of every triangle summed into the global M and K.
// Every global row is an edge (a, b), a < b; all rows of node a -- its larger
// neighbours b -- are enumerated together by one thread from the node's FAN:
// the triangles in which a is the smallest or the middle vertex (exactly the
// triangles holding an edge whose smaller node is a).
//
//   k_fan_fill_fixed     per triangle (p < q < r): one atomic at p and at q,
//                        whose return value is the slot of the triangle id
//                        in the node's C fixed fan slots (C = 4 or 8); two
//                        triangles per thread, one atomic for a shared p
//   k_fan_fallback       only when a fan overflows C (F_FAN_OVER): a scan
//                        of the counts -> fan_ptr and the counting-sort
//                        fill, one launch with grid barriers (it exits at
//                        once otherwise; the plain count / scan / fill
//                        sequence with EFEM_FAN_FIXED=0)
//   k_fan_nodes<FR>      per node: the owned edges as sorted (b, element,
//                        local edge) keys in registers; DOF ids and instance
//                        offsets by a single-pass decoupled look-back over
//                        node tiles; row records, incidence offsets and
//                        elems2dofs in the layout the numeric kernel
//                        k_rows_tri (assemble.cu) reads
//
// Against the bucket pipeline of dofs.cu (instances of all 3 T edges keyed
// by minimum node, 8-byte keys, a count pass and a write pass over them) the
// fans hold 2 T 4-byte triangle ids and one pass over them does the rest
// (DESIGN.md §7).
#include <cub/cub.cuh>

#include <atomic>
#include <type_traits>

#include "efem_internal.cuh"

namespace efem {
namespace {

#ifndef EFEM_FAN_TPB
#define EFEM_FAN_TPB 128
#endif
constexpr int FAN_TPB = EFEM_FAN_TPB;
// Register fast path: fans of <= FR triangles, 2 FR key registers.  FR = 8
// covers every node of the meshes in the tests but one in a thousand; FR = 4
// (all 2D triangulations average 4) leaves registers for 12 CTAs / SM and is
// launched when the previous fan pass of the plan saw no larger fan (a
// larger one then takes the slow path: same result, slower).
constexpr int FAN_REG = 8;
constexpr int FAN_SMALL = 4;
#ifndef EFEM_FAN_MINB
#define EFEM_FAN_MINB 12
#endif
constexpr unsigned long long TS_AGG = 1ull << 62, TS_PRE = 2ull << 62, TS_VAL = (1ull << 62) - 1;

__device__ __forceinline__ bool invalid_node(int v, int64_t n) { return (unsigned long long)(unsigned)v >= (unsigned long long)n; }

__device__ __forceinline__ void sort3(int& p, int& q, int& r) {
    const int a = min(p, q), b = max(p, q);
    p = min(a, r);
    const int m = max(a, r);
    q = min(b, m);
    r = max(b, m);
}

// ---------------------------------------------------------------------------------
// K1 / K2: counting sort of the fan instances (triangle e into the fans of
// its smallest and middle vertex).  The fill takes slots from the top of
// each count (atomicSub), which returns the counts to zero for the next
// call; the order inside a fan is fixed later (ascending e).
// ---------------------------------------------------------------------------------
// (distributed assembly: only the fans of the owned nodes [lo, lo + n_own),
// indexed from lo; single GPU: lo = 0, n_own = n_nodes)
template <bool FILL, bool COH = false>
__device__ __forceinline__ void fan_bucket_one(const int32_t* __restrict__ elems, int64_t e, int64_t n_nodes,
                                               int64_t lo, int64_t n_own, int32_t* __restrict__ cnt,
                                               const int32_t* __restrict__ fan_ptr, int32_t* __restrict__ fan,
                                               WsHeader* hdr) {
    int p = __ldg(elems + 3 * e), q = __ldg(elems + 3 * e + 1), r = __ldg(elems + 3 * e + 2);
    if (invalid_node(p, n_nodes) || invalid_node(q, n_nodes) || invalid_node(r, n_nodes)) {
        if (!FILL) atomicOr(&hdr->flags[F_INVALID_NODE], 1);
        return;  // (skipped consistently by count and fill; the call reports EFEM_EINVAL)
    }
    sort3(p, q, r);
    const int64_t lp = p - lo, lq = q - lo;
    const bool op = (unsigned long long)lp < (unsigned long long)n_own;
    const bool oq = q != p && (unsigned long long)lq < (unsigned long long)n_own;
    if constexpr (!FILL) {
        if (op) atomicAdd(cnt + lp, 1);
        if (oq) atomicAdd(cnt + lq, 1);
    } else {
        // (COH: fan_ptr was written by this kernel's other CTAs: no read-only path)
        if (op) fan[(COH ? __ldcg(fan_ptr + lp) : __ldg(fan_ptr + lp)) + atomicSub(cnt + lp, 1) - 1] = (int)e;
        if (oq) fan[(COH ? __ldcg(fan_ptr + lq) : __ldg(fan_ptr + lq)) + atomicSub(cnt + lq, 1) - 1] = (int)e;
    }
}

template <bool FILL>
__global__ void __launch_bounds__(256) k_fan_bucket(const int32_t* __restrict__ elems, int64_t n_elems, int64_t n_nodes,
                                                    int64_t lo, int64_t n_own, int32_t* __restrict__ cnt,
                                                    const int32_t* __restrict__ fan_ptr, int32_t* __restrict__ fan,
                                                    WsHeader* hdr) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    fan_bucket_one<FILL>(elems, e, n_nodes, lo, n_own, cnt, fan_ptr, fan, hdr);
}

// ---------------------------------------------------------------------------------
// K1' (one pass): fixed-capacity fans, C slots per node -- the atomic's
// return value is the slot, so the count, its scan and the second pass over
// the elements disappear.  A node with more than C fan triangles sets
// F_FAN_OVER; the counting-sort path below then runs on the device (its
// kernels exit at once otherwise), and the fan pass reads its fans instead.
// The counts stay in cnt (zeroed by a memset before the fill: zeroing them
// in the fan pass made its loads wait on the stores, 0.67 -> 1.55 ms; the
// fallback's fill counts them down to zero).
// ---------------------------------------------------------------------------------
// Two consecutive triangles per thread (24 contiguous bytes: three 8-byte
// loads when the element array is 8-byte aligned), all atomics issued
// before the slot stores.  The two triangles of a pair sharing their
// smallest vertex (a structured cell) take both slots with one atomic.
// Slot order inside a fan is immaterial (k_fan_nodes sorts).
template <int C>
__device__ __forceinline__ void fill_put(int32_t* __restrict__ fan_fix, int64_t l, int k, int e, bool& over) {
    if (k < C) fan_fix[l * C + k] = e;
    else over = true;
}
template <int C>
__global__ void __launch_bounds__(256) k_fan_fill_fixed(const int32_t* __restrict__ elems, int64_t n_elems,
                                                         int64_t n_nodes, int64_t lo, int64_t n_own,
                                                         int32_t* __restrict__ cnt, int32_t* __restrict__ fan_fix,
                                                         WsHeader* hdr) {
    const int64_t e0 = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    if (e0 >= n_elems) return;
    int v[6];
    const bool full = e0 + 2 <= n_elems;
    if (full && !(reinterpret_cast<uintptr_t>(elems) & 7)) {
        const int2* p2 = reinterpret_cast<const int2*>(elems + 3 * e0);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const int2 x = __ldg(p2 + q);
            v[2 * q] = x.x;
            v[2 * q + 1] = x.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 6; ++j) v[j] = e0 + j / 3 < n_elems ? __ldg(elems + 3 * e0 + j) : 0;
    }
    bool inval = false;
    bool op[2], oq[2];
    int64_t lp[2], lq[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const bool in = e0 + i < n_elems;
        const bool ok = in && !(invalid_node(v[3 * i], n_nodes) || invalid_node(v[3 * i + 1], n_nodes) ||
                                invalid_node(v[3 * i + 2], n_nodes));
        inval |= in && !ok;
        sort3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
        lp[i] = v[3 * i] - lo;
        lq[i] = v[3 * i + 1] - lo;
        op[i] = ok && (unsigned long long)lp[i] < (unsigned long long)n_own;
        oq[i] = ok && v[3 * i + 1] != v[3 * i] && (unsigned long long)lq[i] < (unsigned long long)n_own;
    }
    if (inval) atomicOr(&hdr->flags[F_INVALID_NODE], 1);
    const bool pair = op[0] && op[1] && lp[0] == lp[1];
    int kp0 = 0, kp1 = 0, kq0 = 0, kq1 = 0, base = 0;
    if (pair) {
        base = atomicAdd(cnt + lp[0], 2);
        kp0 = base;
        kp1 = base + 1;
    } else {
        if (op[0]) kp0 = atomicAdd(cnt + lp[0], 1);
        if (op[1]) kp1 = atomicAdd(cnt + lp[1], 1);
    }
    if (oq[0]) kq0 = atomicAdd(cnt + lq[0], 1);
    if (oq[1]) kq1 = atomicAdd(cnt + lq[1], 1);
    bool over = false;
    if (op[0]) fill_put<C>(fan_fix, lp[0], kp0, (int)e0, over);
    if (op[1]) fill_put<C>(fan_fix, lp[1], kp1, (int)e0 + 1, over);
    if (oq[0]) fill_put<C>(fan_fix, lq[0], kq0, (int)e0, over);
    if (oq[1]) fill_put<C>(fan_fix, lq[1], kq1, (int)e0 + 1, over);
    if (over) atomicOr(&hdr->flags[F_FAN_OVER], 1);
}

// the fallback's scan tiles: 2048 counts
constexpr int CS_TPB = 256, CS_ITEMS = 8, CS_TILE = CS_TPB * CS_ITEMS;

// The whole fallback as ONE launch (a step without an overflow pays one
// launch that exits at once instead of three): the scan's two phases and
// the counting-sort fill separated by software grid barriers.  The grid is
// one CTA per SM, so every CTA is resident (the previous kernel on the
// stream has drained); the barrier counter is the word after the look-back
// tile states, zeroed by k_fan_prep.
__device__ __forceinline__ void fb_grid_sync(unsigned* bar, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (*(volatile unsigned*)bar < target) __nanosleep(100);
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(CS_TPB) k_fan_fallback(const int32_t* __restrict__ elems, int64_t n_elems,
                                                         int64_t n_nodes, int64_t lo, int64_t n_own,
                                                         int32_t* __restrict__ cnt, int32_t* __restrict__ tsum,
                                                         int32_t* __restrict__ fan_ptr, int32_t* __restrict__ fan,
                                                         unsigned* bar, WsHeader* hdr) {
    if (!*(volatile const int*)&hdr->flags[F_FAN_OVER]) return;
    using BS = cub::BlockScan<int, CS_TPB>;
    using BR = cub::BlockReduce<int, CS_TPB>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ typename BR::TempStorage rtmp;
    __shared__ int s_base;
    const int64_t n = n_own;
    const int64_t nt = (n + CS_TILE - 1) / CS_TILE;
    // (1) tile sums of the counts
    for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
        int v = 0;
#pragma unroll
        for (int k = 0; k < CS_ITEMS; ++k) {
            const int64_t i = t * CS_TILE + k * CS_TPB + threadIdx.x;
            if (i < n) v += cnt[i];
        }
        const int sum = BR(rtmp).Sum(v);
        if (threadIdx.x == 0) tsum[t] = sum;
        __syncthreads();
    }
    fb_grid_sync(bar, gridDim.x);
    // (2) exclusive scan of each tile plus the sum of the tile totals before it
    for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
        int v[CS_ITEMS], x[CS_ITEMS];
        const int64_t b = t * CS_TILE + (int64_t)threadIdx.x * CS_ITEMS;  // blocked arrangement
#pragma unroll
        for (int k = 0; k < CS_ITEMS; ++k) v[k] = b + k < n ? cnt[b + k] : 0;
        BS(tmp).ExclusiveSum(v, x);
        int pre = 0;
        for (int64_t q = threadIdx.x; q < t; q += CS_TPB) pre += __ldcg(tsum + q);
        const int bsum = BR(rtmp).Sum(pre);
        if (threadIdx.x == 0) s_base = bsum;
        __syncthreads();
        const int base = s_base;
#pragma unroll
        for (int k = 0; k < CS_ITEMS; ++k)
            if (b + k < n) fan_ptr[b + k] = base + x[k];
        __syncthreads();
    }
    if (blockIdx.x == 0) {  // fan_ptr[n]: the sum of all tile totals
        int pre = 0;
        for (int64_t q = threadIdx.x; q < nt; q += CS_TPB) pre += __ldcg(tsum + q);
        const int tot = BR(rtmp).Sum(pre);
        if (threadIdx.x == 0) fan_ptr[n] = tot;
    }
    fb_grid_sync(bar, 2 * gridDim.x);
    // (3) the counting-sort fill (slots from the top of each count)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_elems; e += (int64_t)gridDim.x * blockDim.x)
        fan_bucket_one<true, true>(elems, e, n_nodes, lo, n_own, cnt, fan_ptr, fan, hdr);
}

// ---------------------------------------------------------------------------------
// K3: per node a, the edges it owns (its distinct larger neighbours b, in
// ascending order: DOF id = first id of the node + rank) and, per edge, the
// fan instances holding it (e << 3 | k, k the local edge of (a, b) in
// triangle e; t <= 2 in a conforming mesh).  Global DOF ids and instance
// offsets come from a single-pass decoupled look-back over node tiles.
// Outputs, in the layout of the bucket pipeline (dofs.cu) that the numeric
// kernel k_rows_tri reads:
//   rec[i]     {first, last} instance of row i (ascending element id)
//   inc_ptr[i] instances of the rows before i (row i starts at i + 2 inc_ptr[i])
//   e2d[3e+k]  DOF id of local edge k of triangle e
// ---------------------------------------------------------------------------------
struct FanNodesArgs {
    const int32_t* elems;
    const int32_t* fan_ptr;  // indexed from node lo
    int32_t* fan;  // big fans (> FAN_REG) are sorted in place here
    int32_t* fan_fix;        // fixed-capacity fans (fix_c slots per node), unless F_FAN_OVER
    int32_t* cnt;            // their counts (returned to zero here)
    int fix_c;               // 0: the counting-sort fans only
    int64_t lo, n_nodes;     // owned nodes [lo, lo + n_nodes)
    int32_t* node_ent;       // optional (n_nodes + 1): first row of each owned node
    int2* rec;
    int32_t* inc_ptr;
    int32_t* e2d;
    unsigned long long* tile_state;
    WsHeader* hdr;
};

__device__ __forceinline__ void load_tri(const int32_t* __restrict__ elems, int e, int& g0, int& g1, int& g2) {
    const int32_t* p = elems + 3 * (int64_t)e;
    g0 = __ldg(p);
    g1 = __ldg(p + 1);
    g2 = __ldg(p + 2);
}

// the owned-edge keys of fan triangle e at node a: (b << 32 | e << 3 | k) for
// each vertex b > a of the triangle, k = the local edge {a, b} (its opposite
// vertex); ~0 when the vertex is not larger than a
__device__ __forceinline__ void tri_keys(int a, int e, int g0, int g1, int g2, unsigned long long& k1,
                                         unsigned long long& k2) {
    const int la = g0 == a ? 0 : (g1 == a ? 1 : 2);
    const int w1 = la == 0 ? 1 : 0, w2 = la == 2 ? 1 : 2;  // the two other positions
    const int v1 = w1 == 0 ? g0 : g1, v2 = w2 == 1 ? g1 : g2;
    const unsigned long long inst1 = (unsigned long long)(((unsigned)e << 3) | (unsigned)(3 - la - w1));
    const unsigned long long inst2 = (unsigned long long)(((unsigned)e << 3) | (unsigned)(3 - la - w2));
    k1 = v1 > a ? ((unsigned long long)(unsigned)v1 << 32) | inst1 : ~0ull;
    k2 = v2 > a ? ((unsigned long long)(unsigned)v2 << 32) | inst2 : ~0ull;
}

// big fan (> FAN_REG instances, rare): insertion sort of the fan in place by
// triangle id; the owned edges are then visited in ascending b by repeated
// minimum scans (quadratic, global memory)
__device__ void fan_sort_inplace(int32_t* f, int n) {
    for (int j = 1; j < n; ++j) {
        const int v = f[j];
        int k = j;
        while (k > 0 && f[k - 1] > v) {
            f[k] = f[k - 1];
            --k;
        }
        f[k] = v;
    }
}

// calls visit(b, first_inst, last_inst, t) for every owned edge (a, b) of the
// big fan f (sorted by element), ascending b
template <class V>
__device__ void fan_edges_slow(const int32_t* __restrict__ elems, const int32_t* f, int a, int n, V&& visit) {
    long long last = a;
    for (;;) {
        int best = INT_MAX;
        for (int j = 0; j < n; ++j) {
            int g0, g1, g2;
            load_tri(elems, f[j], g0, g1, g2);
            unsigned long long k1, k2;
            tri_keys(a, f[j], g0, g1, g2, k1, k2);
            const int b1 = (int)(k1 >> 32), b2 = (int)(k2 >> 32);
            if (k1 != ~0ull && b1 > last && b1 < best) best = b1;
            if (k2 != ~0ull && b2 > last && b2 < best) best = b2;
        }
        if (best == INT_MAX) return;
        int first = -1, lst = -1, t = 0;
        for (int j = 0; j < n; ++j) {  // ascending element id
            int g0, g1, g2;
            load_tri(elems, f[j], g0, g1, g2);
            unsigned long long k1, k2;
            tri_keys(a, f[j], g0, g1, g2, k1, k2);
            for (const unsigned long long k : {k1, k2})
                if (k != ~0ull && (int)(k >> 32) == best) {
                    if (t == 0) first = (int)(unsigned)k;
                    lst = (int)(unsigned)k;
                    ++t;
                }
        }
        visit(best, first, lst, t);
        last = best;
    }
}

constexpr int FAN_REC_STAGE = FAN_TPB * 4;  // staged rows per tile
// register path: one 32-bit key per owned-edge candidate,
//   (b - a) << 5 | j << 2 | k   (j = position in the fan, k = local edge),
// so one sort orders the candidates by b; b - a < 2^27 (else the slow path)
constexpr unsigned KEY_NONE = 0xffffffffu;
constexpr int KEY_DMAX = 1 << 27;

template <int C, int K2>
__device__ __forceinline__ void sort_keys(unsigned (&key)[K2]) {
#pragma unroll
    for (int kk = 2; kk <= C; kk <<= 1)
#pragma unroll
        for (int jj = kk >> 1; jj > 0; jj >>= 1)
#pragma unroll
            for (int x = 0; x < C; ++x) {
                const int y = x ^ jj;
                if (y > x) {
                    const unsigned lo = min(key[x], key[y]), hi = max(key[x], key[y]);
                    const bool asc = (x & kk) == 0;
                    key[x] = asc ? lo : hi;
                    key[y] = asc ? hi : lo;
                }
            }
}

// walk the sorted keys: row(first, last, t) per run of equal b, the run's
// instances e << 3 | k ordered by element
// (sev: the fan's element ids in shared memory, sev[j * FAN_TPB]: one load
// per key instead of a select chain over the register array)
template <int C, int K2, class R>
__device__ __forceinline__ void key_runs(const unsigned (&key)[K2], const int* sev, R&& row) {
    int first = 0, last = 0, t = 0;
    unsigned prev = KEY_NONE;
#pragma unroll
    for (int x = 0; x < C; ++x) {
        const unsigned k = key[x];
        if (k == KEY_NONE) continue;
        const int e = sev[((k >> 2) & 7) * FAN_TPB];
        const int inst = (e << 3) | (int)(k & 3);
        if ((k >> 5) != (prev >> 5)) {
            if (t) row(first, last, t);
            first = last = inst;
            t = 1;
        } else {
            first = min(first, inst);
            last = max(last, inst);
            ++t;
        }
        prev = k;
    }
    if (t) row(first, last, t);
}

#ifndef EFEM_FAN_NPT
#define EFEM_FAN_NPT 1
#endif
#ifndef EFEM_FAN_MINB2
#define EFEM_FAN_MINB2 8
#endif
constexpr int FAN_NPT = EFEM_FAN_NPT;  // owned nodes per thread (blocked: thread x holds nodes NPT x .. NPT x + NPT - 1)
constexpr int FAN_TILE = FAN_TPB * FAN_NPT;

template <int FR>
__global__ void __launch_bounds__(FAN_TPB, FAN_NPT == 1 ? EFEM_FAN_MINB : EFEM_FAN_MINB2) k_fan_nodes(FanNodesArgs A) {
    constexpr int NPT = FAN_NPT;
    using BlockScan = cub::BlockScan<unsigned long long, FAN_TPB, cub::BLOCK_SCAN_WARP_SCANS>;
    __shared__ typename BlockScan::TempStorage scan_tmp;
    __shared__ unsigned long long s_excl;
    __shared__ int2 s_rec[FAN_REC_STAGE * NPT];
    __shared__ int s_inc[FAN_REC_STAGE * NPT];
    __shared__ int s_ev[NPT * FR * FAN_TPB];  // the fans' element ids, [(h FR + j) FAN_TPB + thread]
    // tiles in launch order (CTAs are dispatched in blockIdx order, so every
    // predecessor a tile waits on is resident or done -- as CUB's single-pass
    // scans); the overflow flag through the read-only path (one L1 line per
    // SM): no ticket round trip and no barrier before the loads
    const int tile = blockIdx.x;
    const bool csr = A.fix_c == 0 || __ldg(&A.hdr->flags[F_FAN_OVER]);
    const int64_t l0 = (int64_t)tile * FAN_TILE + (int64_t)threadIdx.x * NPT;  // first owned node index
    int n_ent[NPT], n_inst[NPT], beg[NPT], n[NPT];
    bool slow[NPT];
    bool bad = false, big = false;
    unsigned key[NPT][2 * FR];
    int ev[NPT][FR];
#pragma unroll
    for (int h = 0; h < NPT; ++h) {
        n_ent[h] = n_inst[h] = beg[h] = n[h] = 0;
        slow[h] = false;
#pragma unroll
        for (int x = 0; x < 2 * FR; ++x) key[h][x] = KEY_NONE;
#pragma unroll
        for (int j = 0; j < FR; ++j) ev[h][j] = 0;
    }
    int32_t* const fbase = csr ? A.fan : A.fan_fix;
    // fixed slots of this launch's width: all FR slots as 16-byte loads,
    // issued with the count load (slots past the count are ignored)
    const bool vec = !csr && A.fix_c == FR;
#pragma unroll
    for (int h = 0; h < NPT; ++h) {
        const int64_t l64 = l0 + h;
        if (l64 < A.n_nodes) {
            if (vec) {
                const int4* p4 = reinterpret_cast<const int4*>(A.fan_fix + l64 * FR);
#pragma unroll
                for (int q = 0; q < FR / 4; ++q) {
                    const int4 v = __ldg(p4 + q);
                    ev[h][4 * q] = v.x;
                    ev[h][4 * q + 1] = v.y;
                    ev[h][4 * q + 2] = v.z;
                    ev[h][4 * q + 3] = v.w;
                }
            }
            if (csr) {
                beg[h] = __ldg(A.fan_ptr + l64);
                n[h] = __ldg(A.fan_ptr + l64 + 1) - beg[h];
            } else {
                beg[h] = (int)l64 * A.fix_c;
                n[h] = __ldg(A.cnt + l64);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < NPT; ++h) {
        const int64_t l64 = l0 + h;
        if (l64 >= A.n_nodes) continue;
        const int a = (int)(A.lo + l64);
        const int nh = n[h];
        slow[h] = nh > FR;
        big |= nh > FAN_SMALL;  // (for the next launch's choice of FR)
        if (!slow[h]) {
            if (!vec) {
#pragma unroll
                for (int j = 0; j < FR; ++j) ev[h][j] = j < nh ? fbase[beg[h] + j] : 0;
            }
#pragma unroll
            for (int j = 0; j < FR; ++j)
                if (j < nh) s_ev[(h * FR + j) * FAN_TPB + threadIdx.x] = ev[h][j];
#pragma unroll
            for (int j = 0; j < FR; ++j) {
                if (j < nh) {
                    int g0, g1, g2;
                    load_tri(A.elems, ev[h][j], g0, g1, g2);
                    const int la = g0 == a ? 0 : (g1 == a ? 1 : 2);
                    const int w1 = la == 0 ? 1 : 0, w2 = la == 2 ? 1 : 2;  // the two other positions
                    const int v1 = w1 == 0 ? g0 : g1, v2 = w2 == 1 ? g1 : g2;
                    // (a vertex id above a by 2^27 or more takes the slow path)
                    slow[h] |= (v1 > a && v1 - a >= KEY_DMAX) || (v2 > a && v2 - a >= KEY_DMAX);
                    if (v1 > a) key[h][2 * j] = ((unsigned)(v1 - a) << 5) | (j << 2) | (unsigned)(3 - la - w1);
                    if (v2 > a) key[h][2 * j + 1] = ((unsigned)(v2 - a) << 5) | (j << 2) | (unsigned)(3 - la - w2);
                }
            }
        }
        if (!slow[h]) {
            auto count = [&](auto cmax) {
                constexpr int CM = decltype(cmax)::value;
                sort_keys<CM>(key[h]);
#pragma unroll
                for (int x = 0; x < CM; ++x) {
                    const bool v = key[h][x] != KEY_NONE;
                    n_inst[h] += v;
                    n_ent[h] += v && (x == 0 || (key[h][x] >> 5) != (key[h][x - 1] >> 5));
                    if (x >= 2) bad |= v && (key[h][x] >> 5) == (key[h][x - 2] >> 5);  // an edge in three triangles
                }
            };
            if (nh <= FR / 2) count(std::integral_constant<int, FR>{});
            else count(std::integral_constant<int, 2 * FR>{});
        } else {
            fan_sort_inplace(fbase + beg[h], nh);
            fan_edges_slow(A.elems, fbase + beg[h], a, nh, [&](int, int, int, int t) {
                ++n_ent[h];
                n_inst[h] += t;
                bad |= t > 2;
            });
        }
    }
    if (bad) atomicOr(&A.hdr->flags[F_ROW_MISMATCH], 1);
    // tile prefix of (entities << 31 | instances)
    unsigned long long mine[NPT], off[NPT], agg;
#pragma unroll
    for (int h = 0; h < NPT; ++h) mine[h] = ((unsigned long long)n_ent[h] << 31) | (unsigned long long)n_inst[h];
    BlockScan(scan_tmp).ExclusiveSum(mine, off, agg);
    if (threadIdx.x < 32) {
        // decoupled look-back (warp 0): publish the aggregate, sum the
        // predecessors' aggregates back to the nearest inclusive prefix
        unsigned long long excl = 0;
        if (tile == 0) {
            if (threadIdx.x == 0) atomicExch(A.tile_state, TS_PRE | agg);
        } else {
            if (threadIdx.x == 0) atomicExch(A.tile_state + tile, TS_AGG | agg);
            int j = tile - 1;
            for (;;) {
                const int idx = j - (int)threadIdx.x;
                unsigned long long st = TS_PRE;  // (before tile 0: an empty prefix)
                if (idx >= 0) {
                    do {
                        st = *(volatile unsigned long long*)(A.tile_state + idx);
                    } while ((st >> 62) == 0);
                }
                const unsigned pre = __ballot_sync(0xffffffffu, (st >> 62) == 2);
                const int stop = pre ? __ffs(pre) - 1 : 32;  // nearest lane with an inclusive prefix
                unsigned long long v = (int)threadIdx.x <= stop ? (st & TS_VAL) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                excl += v;
                if (pre) break;
                j -= 32;
            }
            if (threadIdx.x == 0) atomicExch(A.tile_state + tile, TS_PRE | (excl + agg));
        }
        if (threadIdx.x == 0) s_excl = excl;
    }
    __syncthreads();
    if (__any_sync(0xffffffffu, big) && (threadIdx.x & 31) == 0 && !__ldg(&A.hdr->fan_big))
        atomicOr(&A.hdr->fan_big, 1);
    const unsigned long long base = s_excl;
    const int e_tile0 = (int)(base >> 31), i_tile0 = (int)(base & 0x7fffffffull);
    const int e_tot = (int)(agg >> 31);
    const bool stage = e_tot <= FAN_REC_STAGE * NPT;
#pragma unroll
    for (int h = 0; h < NPT; ++h) {
        const int64_t l64 = l0 + h;
        if (l64 >= A.n_nodes) continue;
        const int a = (int)(A.lo + l64);
        int id = e_tile0 + (int)(off[h] >> 31);  // first DOF of node a
        int inst = i_tile0 + (int)(off[h] & 0x7fffffffull);
        if (A.node_ent) A.node_ent[l64] = id;
        auto row = [&](int first, int last, int t) {
            if (stage) {
                s_rec[id - e_tile0] = make_int2(first, last);
                s_inc[id - e_tile0] = inst;
            } else {
                A.rec[id] = make_int2(first, last);
                A.inc_ptr[id] = inst;
            }
            A.e2d[(int64_t)(first >> 3) * 3 + (first & 7)] = id;
            if (t > 1) A.e2d[(int64_t)(last >> 3) * 3 + (last & 7)] = id;
            ++id;
            inst += t;
        };
        if (!slow[h]) {
            const int* sev = s_ev + h * FR * FAN_TPB + threadIdx.x;
            if (n[h] <= FR / 2) key_runs<FR>(key[h], sev, row);
            else key_runs<2 * FR>(key[h], sev, row);
        } else {
            fan_edges_slow(A.elems, fbase + beg[h], a, n[h],
                           [&](int, int first, int last, int t) { row(first, last, min(t, 2)); });
        }
        if (l64 == A.n_nodes - 1) {
            if (A.node_ent) A.node_ent[A.n_nodes] = id;
            A.inc_ptr[id] = inst;
            A.hdr->totals[0] = id;
            A.hdr->totals[1] = (long long)id + 2ll * inst;  // sum_i (1 + 2 t_i)
        }
    }
    if (stage) {
        __syncthreads();
        for (int x = threadIdx.x; x < e_tot; x += FAN_TPB) {
            A.rec[e_tile0 + x] = s_rec[x];
            A.inc_ptr[e_tile0 + x] = s_inc[x];
        }
    }
}

}  // namespace

namespace {
__global__ void k_fan_init(WsHeader* hdr) {
    const int i = threadIdx.x;
    if (i < F_NFLAGS) hdr->flags[i] = 0;
    if (i == 0) {
        hdr->bad_element = ~0ull;
        hdr->totals[0] = 0;
        hdr->totals[1] = 0;
        hdr->fan_big = 0;
    }
}

// one launch before the fill: header reset (reset != 0), the fan counts and
// the look-back tile states zeroed (in place of two memsets)
__global__ void __launch_bounds__(256) k_fan_prep(WsHeader* hdr, int reset, int32_t* __restrict__ cnt, int64_t n,
                                                  unsigned long long* __restrict__ tiles, int64_t ntiles) {
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
    if (reset && blockIdx.x == 0) {
        const int i = threadIdx.x;
        if (i < F_NFLAGS) hdr->flags[i] = 0;
        if (i == 0) {
            hdr->bad_element = ~0ull;
            hdr->totals[0] = 0;
            hdr->totals[1] = 0;
            hdr->fan_big = 0;
        }
    }
    const int64_t n4 = n >> 2;  // (cnt is 256-byte aligned: int4 stores)
    int4* c4 = reinterpret_cast<int4*>(cnt);
    for (int64_t i = i0; i < n4; i += st) c4[i] = make_int4(0, 0, 0, 0);
    for (int64_t i = 4 * n4 + i0; i < n; i += st) cnt[i] = 0;
    for (int64_t i = i0; i < ntiles; i += st) tiles[i] = 0ull;
}

}  // namespace

// The symbolic half (K1-K3): sizes in the header totals, offsets and
// neighbour lists in the plan's fan arrays.  Enqueue only.
efem_status launch_hdr_reset(Plan& p, cudaStream_t s) {
    k_fan_init<<<1, 32, 0, s>>>(p.hdr);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

efem_status launch_fan_symbolic(Plan& p, cudaStream_t s, bool reset) {
    const int64_t Ng = p.n_nodes, T = p.n_elems;
    const int64_t lo = p.own_lo, N = p.own_n < 0 ? Ng : p.own_n;  // owned nodes [lo, lo + N)
#ifndef EFEM_FAN_FIXED
#define EFEM_FAN_FIXED 1
#endif
    // fixed-capacity fill (4 slots when the plan's last fan pass saw no fan
    // above 4, else 8) with the counting sort as the on-device fallback
    const int fix_c = EFEM_FAN_FIXED ? (p.fan_small ? 4 : FAN_FIXC) : 0;
    const int ntiles = (int)grid_for(N, FAN_TILE);
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (fix_c) {
        const int64_t work = std::max<int64_t>(N / 4, ntiles);
        const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(work, 256), 8 * sms));
        k_fan_prep<<<g, 256, 0, s>>>(p.hdr, reset ? 1 : 0, p.cnt, N, p.fan_tiles, ntiles + 1);  // (+ the fallback's barrier word)
        EFEM_LAUNCH_CHECK();
    } else {
        if (reset) {
            k_fan_init<<<1, 32, 0, s>>>(p.hdr);
            EFEM_LAUNCH_CHECK();
        }
        if (ntiles > 0) EFEM_CUDA_TRY(cudaMemsetAsync(p.fan_tiles, 0, (size_t)ntiles * 8, s));
    }
    if (fix_c) {
        if (T > 0) {
            if (fix_c == 4)
                k_fan_fill_fixed<4><<<grid_for((T + 1) / 2, 256), 256, 0, s>>>(p.elems, T, Ng, lo, N, p.cnt, p.fan_fix,
                                                                                p.hdr);
            else
                k_fan_fill_fixed<FAN_FIXC><<<grid_for((T + 1) / 2, 256), 256, 0, s>>>(p.elems, T, Ng, lo, N, p.cnt, p.fan_fix,
                                                                              p.hdr);
            EFEM_LAUNCH_CHECK();
        }
        k_fan_fallback<<<sms, CS_TPB, 0, s>>>(p.elems, T, Ng, lo, N, p.cnt, p.fan_csum, p.fan_ptr, p.fan,
                                              reinterpret_cast<unsigned*>(p.fan_tiles + ntiles), p.hdr);
        EFEM_LAUNCH_CHECK();
    } else {
        if (T > 0) {
            k_fan_bucket<false><<<grid_for(T, 256), 256, 0, s>>>(p.elems, T, Ng, lo, N, p.cnt, nullptr, nullptr,
                                                                 p.hdr);
            EFEM_LAUNCH_CHECK();
        }
        size_t bytes = p.cub_bytes;
        EFEM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(p.cub_tmp, bytes, p.cnt, p.fan_ptr, (int)(N + 1), s));
        count_launch(2);
        if (T > 0) {
            k_fan_bucket<true><<<grid_for(T, 256), 256, 0, s>>>(p.elems, T, Ng, lo, N, p.cnt, p.fan_ptr, p.fan, p.hdr);
            EFEM_LAUNCH_CHECK();
        }
    }
    if (N == 0) {  // no owned node: an empty row set
        EFEM_CUDA_TRY(cudaMemsetAsync(p.inc_ptr, 0, 4, s));
        if (p.node_ent) EFEM_CUDA_TRY(cudaMemsetAsync(p.node_ent, 0, 4, s));
        return EFEM_OK;
    }
    FanNodesArgs A{p.elems, p.fan_ptr, p.fan, p.fan_fix, p.cnt, fix_c, lo, N, p.node_ent, p.rec, p.inc_ptr, p.e2d,
                   p.fan_tiles, p.hdr};
    if (p.fan_small) k_fan_nodes<FAN_SMALL><<<ntiles, FAN_TPB, 0, s>>>(A);
    else k_fan_nodes<FAN_REG><<<ntiles, FAN_TPB, 0, s>>>(A);
    EFEM_LAUNCH_CHECK();
    return EFEM_OK;
}

size_t fan_tiles_bytes(int64_t n_nodes) { return ((size_t)(n_nodes + FAN_TPB - 1) / FAN_TPB + 1) * 8; }

}  // namespace efem
