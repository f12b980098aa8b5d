// common.cuh — device primitives shared by the C-SAW kernels (sm_100a).
//
// Counter-based Philox4x32-10 draws (reading R7), below(U, M), and warp-level
// scan / reduce / sort helpers built on __shfl*_sync, __ballot_sync and
// __match_any_sync.  This file is independent of oracle/ (no shared code).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#ifdef CSAW_DEBUG_BOUNDS
#include <cstdio>
#endif

namespace csaw {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr uint32_t NONE = 0xFFFFFFFFu;

// Purposes of a draw (counter word 3, bits 28..31).
enum : uint32_t { PURPOSE_EDGE = 0, PURPOSE_VERTEX = 1, PURPOSE_BURN = 2, PURPOSE_ACCEPT = 3, PURPOSE_JUMP = 4,
                  PURPOSE_TARGET = 5 };

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Philox4x32-10 (Salmon et al., SC'11).  10 rounds of two 32x32->64 multiplies.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ uint2 philox_key(uint64_t seed) {
    return make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

__device__ __forceinline__ uint32_t word3(uint32_t purpose, uint32_t j, uint32_t a) {
    return (purpose << 28) | (j << 14) | a;
}

// U = o0 | o1 << 32 of philox((inst, t, slot, w3); key).
__device__ __forceinline__ uint64_t draw_u64(uint2 key, uint32_t inst, uint32_t t, uint32_t slot, uint32_t w3) {
    const uint4 o = philox4x32_10(make_uint4(inst, t, slot, w3), key);
    return static_cast<uint64_t>(o.x) | (static_cast<uint64_t>(o.y) << 32);
}

// below(U, M) = floor(U * M / 2^64), uniform in [0, M).
__device__ __forceinline__ uint64_t below(uint64_t U, uint64_t M) { return __umul64hi(U, M); }

// Device bounds checks of a debug build (-DCSAW_DEBUG_BOUNDS: scripts/build_variants.sh); no code otherwise.
#ifdef CSAW_DEBUG_BOUNDS
#define CSAW_DASSERT(cond)                                                                      \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("CSAW_DASSERT failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);            \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define CSAW_DASSERT(cond) ((void)0)
#endif

// ---------------------------------------------------------------- random single-word loads
// An L2 miss of a lone 4 / 8 B load fetches a whole 128 B line (4 sectors) from DRAM by
// default; the .L2::64B prefetch-size qualifier (SASS LDG.E.LTC64B) limits it to 64 B.
// Measured on B200 (scripts/random_granule.cu, profiles/r02_random_granule.txt): 127 -> 64 DRAM
// bytes per random 4 B read at the same ~35 G reads/s.  For the pointer-chasing loads whose
// neighbours are never used (the MDRW per-step entry / metadata / vertex-id reads; the node2vec
// index probes keep whole lines: .L2::64B there measured 7.81 vs 7.54 ms on cfg3).
#ifndef CSAW_LD64B
#define CSAW_LD64B 1
#endif
// coherent (not .nc) variant for state the kernel itself writes
__device__ __forceinline__ uint32_t ld_rand_rw_u32(const uint32_t* p) {
#if CSAW_LD64B
    uint32_t v;
    asm volatile("ld.global.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
#else
    return *p;
#endif
}
// evict-first variants (read-once streams that should not displace reused state)
__device__ __forceinline__ uint32_t ld_rand_cs_u32(const uint32_t* p) {
#if CSAW_LD64B
    uint32_t v;
    asm("ld.global.cs.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#else
    return __ldcs(p);
#endif
}
__device__ __forceinline__ uint64_t ld_rand_cs_u64(const uint64_t* p) {
#if CSAW_LD64B
    uint64_t v;
    asm("ld.global.cs.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
#else
    return __ldcs(p);
#endif
}
__device__ __forceinline__ uint4 ld_rand_cs_v4(const uint4* p) {
#if CSAW_LD64B
    uint4 v;
    asm("ld.global.cs.L2::64B.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
#else
    return __ldcs(p);
#endif
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t v) {
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) { return __reduce_max_sync(FULL, v); }

// Ascending bitonic sort of one u32 per lane across the warp.
__device__ __forceinline__ uint32_t warp_sort_u32(uint32_t v) {
    const int lane = lane_id();
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint32_t o = __shfl_xor_sync(FULL, v, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            v = (lower == up) ? min(v, o) : max(v, o);
        }
    }
    return v;
}

// First index in sorted a[lo, hi) with a[idx] >= key (hi if none).  Warp-collective
// 32-ary search: one round of 32 parallel probes shrinks the range 32x.
__device__ __forceinline__ uint64_t warp_lower_bound(const uint32_t* __restrict__ a, uint64_t lo, uint64_t hi,
                                                     uint32_t key) {
    const int lane = lane_id();
    while (hi - lo > 32) {
        const uint64_t step = (hi - lo + 31) / 32;
        const uint64_t p = lo + static_cast<uint64_t>(lane) * step;
        const bool ok = p < hi && __ldg(a + p) >= key;
        const unsigned b = __ballot_sync(FULL, ok);
        const unsigned inb = __ballot_sync(FULL, p < hi);
        if (b == 0) {
            const int last = 31 - __clz(inb);
            lo = lo + static_cast<uint64_t>(last) * step + 1;
        } else {
            const int f = __ffs(b) - 1;
            if (f == 0) return lo;
            const uint64_t pf = lo + static_cast<uint64_t>(f) * step;
            lo = lo + static_cast<uint64_t>(f - 1) * step + 1;
            hi = pf;
        }
    }
    const uint64_t p = lo + lane;
    const bool ok = p < hi && __ldg(a + p) >= key;
    const unsigned b = __ballot_sync(FULL, ok);
    return b ? lo + (__ffs(b) - 1) : hi;
}

// First index in a[lo, hi) with a[idx] > x (hi if none), for a sorted non-decreasing u64
// array.  Warp-collective 32-ary search: ceil(log32(hi - lo)) rounds of 32 parallel
// probes (one round trip each) instead of log2 dependent loads.  *probes counts loads.
__device__ __forceinline__ uint64_t warp_upper_bound_u64(const uint64_t* __restrict__ a, uint64_t lo, uint64_t hi,
                                                         uint64_t x, uint32_t* probes) {
    const int lane = lane_id();
    while (hi - lo > 32) {
        const uint64_t step = (hi - lo + 31) / 32;
        const uint64_t p = lo + static_cast<uint64_t>(lane) * step;
        const bool inr = p < hi;
        const bool ok = inr && __ldg(a + p) > x;
        const unsigned b = __ballot_sync(FULL, ok);
        const unsigned inb = __ballot_sync(FULL, inr);
        *probes += __popc(inb);
        if (b == 0) {
            const int last = 31 - __clz(inb);
            lo = lo + static_cast<uint64_t>(last) * step + 1;
        } else {
            const int f = __ffs(b) - 1;
            if (f == 0) return lo;
            const uint64_t pf = lo + static_cast<uint64_t>(f) * step;
            lo = lo + static_cast<uint64_t>(f - 1) * step + 1;
            hi = pf;
        }
    }
    const uint64_t p = lo + lane;
    const bool ok = p < hi && __ldg(a + p) > x;
    *probes += static_cast<uint32_t>(min(static_cast<uint64_t>(32), hi - lo));
    const unsigned b = __ballot_sync(FULL, ok);
    return b ? lo + (__ffs(b) - 1) : hi;
}

// Grid helpers
__device__ __forceinline__ uint64_t global_warp_id() {
    return (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
}
__device__ __forceinline__ uint64_t total_warps() {
    return (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
}

}  // namespace csaw
