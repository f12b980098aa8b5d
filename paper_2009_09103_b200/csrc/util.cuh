// util.cuh — device-wide exclusive scan and stable LSD radix sort (own kernels).
//
// Used by the traversal-sampling driver for output offsets, frontier-queue
// compaction and the per-instance frontier dedup (sorting (instance, vertex)
// keys).  Sizes are host-known; every kernel is a grid-stride or fixed-grid
// launch on the caller's stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace csaw {

constexpr int SCAN_BLOCK = 1024;
constexpr int SCAN_MAX_GRID = 1024;

// ---------------------------------------------------------------- block scan
template <int NT>
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t* wsum, uint64_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t incl = warp_incl_scan(v);
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        const uint64_t x = lane < NT / 32 ? wsum[lane] : 0;
        const uint64_t xi = warp_incl_scan(x);
        if (lane < NT / 32) wsum[lane] = xi - x;
        if (lane == NT / 32 - 1) *total = xi;
    }
    __syncthreads();
    const uint64_t r = wsum[w] + incl - v;
    __syncthreads();
    return r;
}

// Val: functor uint64 operator()(uint64 i) for i < n.
template <class Val>
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_partials(Val val, uint64_t n, uint64_t chunk, uint64_t* part) {
    __shared__ uint64_t wsum[SCAN_BLOCK / 32];
    const uint64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    uint64_t s = 0;
    for (uint64_t i = b0 + threadIdx.x; i < b1; i += SCAN_BLOCK) s += val(i);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint64_t t = threadIdx.x < SCAN_BLOCK / 32 ? wsum[threadIdx.x] : 0;
        t = warp_sum(t);
        if (threadIdx.x == 0) part[blockIdx.x] = t;
    }
}

static __global__ void __launch_bounds__(SCAN_BLOCK) k_scan_top(uint64_t* part, int g) {
    __shared__ uint64_t wsum[SCAN_BLOCK / 32];
    __shared__ uint64_t total;
    const uint64_t v = threadIdx.x < g ? part[threadIdx.x] : 0;
    const uint64_t e = block_excl_scan<SCAN_BLOCK>(v, wsum, &total);
    if (threadIdx.x < g) part[threadIdx.x] = e;
    if (threadIdx.x == 0) part[g] = total;
}

template <class Val, class Out>
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_final(Val val, uint64_t n, uint64_t chunk, const uint64_t* part,
                                                           int g, Out out) {
    __shared__ uint64_t wsum[SCAN_BLOCK / 32];
    __shared__ uint64_t total;
    const uint64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    uint64_t carry = part[blockIdx.x];
    for (uint64_t t0 = b0; t0 < b1; t0 += SCAN_BLOCK) {
        const uint64_t i = t0 + threadIdx.x;
        const uint64_t v = i < b1 ? val(i) : 0;
        const uint64_t e = block_excl_scan<SCAN_BLOCK>(v, wsum, &total);
        if (i < b1) out(i, carry + e, v);
        carry += total;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out.total(n, part[g]);
}

// Writes exclusive prefix sums to dst[0..n) and the total to dst[n].
struct ScanToArray {
    uint64_t* dst;
    __device__ __forceinline__ void operator()(uint64_t i, uint64_t e, uint64_t) const { dst[i] = e; }
    __device__ __forceinline__ void total(uint64_t n, uint64_t t) const { dst[n] = t; }
};

// Small n (<= SCAN_BLOCK * SCAN_ONE_PER): one block, each thread a contiguous run of
// ceil(n / SCAN_BLOCK) values -> one launch instead of three.
constexpr uint64_t SCAN_ONE_PER = 32;
template <class Val, class Out>
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_one(Val val, uint64_t n, Out out) {
    __shared__ uint64_t wsum[SCAN_BLOCK / 32];
    __shared__ uint64_t total;
    const uint64_t per = (n + SCAN_BLOCK - 1) / SCAN_BLOCK;
    const uint64_t b0 = min(n, threadIdx.x * per), b1 = min(n, b0 + per);
    uint64_t s = 0;
    for (uint64_t i = b0; i < b1; ++i) s += val(i);
    uint64_t run = block_excl_scan<SCAN_BLOCK>(s, wsum, &total);
    for (uint64_t i = b0; i < b1; ++i) {
        const uint64_t v = val(i);
        out(i, run, v);
        run += v;
    }
    if (threadIdx.x == 0) out.total(n, total);
}

// Host driver: exclusive scan of val(0..n) -> out; part = device scratch >= SCAN_MAX_GRID+1 u64.
template <class Val, class Out>
csaw_status device_scan(Val val, uint64_t n, Out out, uint64_t* part, cudaStream_t st) {
    if (n > 0 && n <= SCAN_BLOCK * SCAN_ONE_PER) {
        k_scan_one<<<1, SCAN_BLOCK, 0, st>>>(val, n, out);
        note_launch();
        CSAW_CUDA(cudaGetLastError());
        return CSAW_OK;
    }
    int g = static_cast<int>(std::min<uint64_t>(SCAN_MAX_GRID, (n + 8 * SCAN_BLOCK - 1) / (8 * SCAN_BLOCK)));
    if (g < 1) g = 1;
    const uint64_t chunk = (n + g - 1) / g;
    if (n > 0) { k_scan_partials<<<g, SCAN_BLOCK, 0, st>>>(val, n, chunk, part); note_launch(); }
    else CSAW_CUDA(cudaMemsetAsync(part, 0, sizeof(uint64_t) * g, st));
    k_scan_top<<<1, SCAN_BLOCK, 0, st>>>(part, g);
    k_scan_final<<<g, SCAN_BLOCK, 0, st>>>(val, n, chunk, part, g, out);
    note_launch(2);
    CSAW_CUDA(cudaGetLastError());
    return CSAW_OK;
}

// ---------------------------------------------------------------- radix sort (u64 keys, stable, LSD 8-bit)
constexpr int RS_BLOCK = 256;
constexpr int RS_WARPS = RS_BLOCK / 32;

static __global__ void __launch_bounds__(RS_BLOCK) k_rs_hist(const uint64_t* __restrict__ keys, uint64_t n, uint64_t chunk,
                                                      int shift, uint64_t* __restrict__ hist, int g) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    for (uint64_t i = b0 + threadIdx.x; i < b1; i += RS_BLOCK) atomicAdd(&h[(keys[i] >> shift) & 255], 1u);
    __syncthreads();
    hist[static_cast<uint64_t>(threadIdx.x) * g + blockIdx.x] = h[threadIdx.x];   // digit-major
}

static __global__ void __launch_bounds__(RS_BLOCK) k_rs_scatter(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                         uint64_t n, uint64_t chunk, int shift,
                                                         const uint64_t* __restrict__ offs, int g) {
    __shared__ uint32_t wcnt[RS_WARPS][256];
    __shared__ uint64_t running[256];
    __shared__ uint32_t tile_tot[256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    running[threadIdx.x] = offs[static_cast<uint64_t>(threadIdx.x) * g + blockIdx.x];
    const uint64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    for (uint64_t t0 = b0; t0 < b1; t0 += RS_BLOCK) {
#pragma unroll
        for (int q = 0; q < RS_WARPS; ++q) wcnt[q][threadIdx.x] = 0;
        __syncthreads();
        const uint64_t i = t0 + threadIdx.x;
        const bool valid = i < b1;
        const uint64_t k = valid ? in[i] : 0;
        const uint32_t dg = valid ? static_cast<uint32_t>((k >> shift) & 255) : 256u;
        const unsigned peers = __match_any_sync(FULL, dg);
        const uint32_t rank = __popc(peers & lanemask_lt());
        if (valid && rank == 0) wcnt[w][dg] = __popc(peers);
        __syncthreads();
        {   // exclusive scan over warps for digit threadIdx.x
            uint32_t acc = 0;
#pragma unroll
            for (int q = 0; q < RS_WARPS; ++q) {
                const uint32_t c = wcnt[q][threadIdx.x];
                wcnt[q][threadIdx.x] = acc;
                acc += c;
            }
            tile_tot[threadIdx.x] = acc;
        }
        __syncthreads();
        if (valid) out[running[dg] + wcnt[w][dg] + rank] = k;
        __syncthreads();
        running[threadIdx.x] += tile_tot[threadIdx.x];
        __syncthreads();
    }
    (void)lane;
}

struct HistVal {
    const uint64_t* h;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return h[i]; }
};

// Sorts keys[0..n) on bits [0, nbits); result pointer returned in *sorted (keys or alt).
inline csaw_status radix_sort_u64(uint64_t* keys, uint64_t* alt, uint64_t n, int nbits, uint64_t* hist,
                                  uint64_t* hoffs, uint64_t* part, uint64_t** sorted, cudaStream_t st) {
    int g = static_cast<int>(std::min<uint64_t>(512, (n + 4095) / 4096));
    if (g < 1) g = 1;
    const uint64_t chunk = (n + g - 1) / g;
    uint64_t* a = keys;
    uint64_t* b = alt;
    if (n > 1) {
        for (int shift = 0; shift < nbits; shift += 8) {
            k_rs_hist<<<g, RS_BLOCK, 0, st>>>(a, n, chunk, shift, hist, g);
            CSAW_TRY(device_scan(HistVal{hist}, static_cast<uint64_t>(256) * g, ScanToArray{hoffs}, part, st));
            k_rs_scatter<<<g, RS_BLOCK, 0, st>>>(a, b, n, chunk, shift, hoffs, g);
            note_launch(2);
            uint64_t* t = a; a = b; b = t;
        }
        CSAW_CUDA(cudaGetLastError());
    }
    *sorted = a;
    return CSAW_OK;
}

inline int bits_for(uint64_t maxval) {
    int b = 0;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return b;
}

}  // namespace csaw
