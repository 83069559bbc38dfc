// scan.cuh -- single-pass block scan + decoupled look-back over CTA tiles.
//
// Used to turn per-node counts (entities owned, CSR entries of their rows)
// into global offsets inside the kernel that produced the counts, so the
// enumeration needs no separate count / scan / fill passes.  Tiles are taken
// in launch order from an atomic ticket, so every predecessor tile is already
// resident when a tile looks back (no deadlock).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace efem {

constexpr unsigned long long LB_FLAG_A = 1ull << 62;  // aggregate published
constexpr unsigned long long LB_FLAG_P = 2ull << 62;  // inclusive prefix published
constexpr unsigned long long LB_VALUE = (1ull << 62) - 1ull;

__device__ __forceinline__ void lb_store(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Called by ALL 32 lanes of ONE warp of the tile (warp-parallel look-back:
// 32 predecessors per step, CUB-style).  Returns the tile's exclusive prefix
// in every lane.  `agg` must be < 2^62.
__device__ __forceinline__ unsigned long long lookback(unsigned long long* status, int tile,
                                                       unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) lb_store(status, LB_FLAG_P | agg);
        return 0ull;
    }
    if (lane == 0) lb_store(status + tile, LB_FLAG_A | agg);
    unsigned long long prefix = 0ull;
    int end = tile - 1;  // nearest predecessor of the current window
    while (true) {
        const int j = end - lane;
        const unsigned long long s = j >= 0 ? lb_load(status + j) : LB_FLAG_P;  // virtual P(0) before tile 0
        const unsigned long long f = s & ~LB_VALUE;
        if (__any_sync(0xffffffffu, f == 0ull)) continue;  // window not fully published yet
        const unsigned pmask = __ballot_sync(0xffffffffu, f == LB_FLAG_P);
        const int stop = pmask ? __ffs(pmask) - 1 : 31;
        unsigned long long v = lane <= stop ? (s & LB_VALUE) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        prefix += v;
        if (pmask) break;
        end -= 32;
    }
    if (lane == 0) lb_store(status + tile, LB_FLAG_P | (prefix + agg));
    return prefix;
}

// Exclusive block scan of one 64-bit value per thread (blockDim.x == TPB,
// multiple of 32).  Returns this thread's exclusive prefix; *total = block sum.
template <int TPB>
__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long v, unsigned long long* total,
                                                                   unsigned long long* smem /* TPB/32 + 1 */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0ull;
        for (int w = 0; w < TPB / 32; ++w) {
            const unsigned long long t = smem[w];
            smem[w] = run;
            run += t;
        }
        smem[TPB / 32] = run;
    }
    __syncthreads();
    *total = smem[TPB / 32];
    return smem[warp] + x - v;
}

}  // namespace efem
