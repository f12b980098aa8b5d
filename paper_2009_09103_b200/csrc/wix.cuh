// wix.cuh — narrow walk index over the static-bias CTPS cache (NEXT-1).
//
// A degree-biased walk step is latency-bound: 4,000 walkers each run a serial
// chain of dependent loads (row -> index levels -> leaf + col -> next row), so
// the number of round trips per step and the instructions between them set the
// speed, not bytes.  This index cuts both against the fanout-32 u64 B-tree of
// select.cuh (CpsTree):
//   * every row total T < 2^32 (checked at build), so S fits u32: a 128-entry
//     internal node is one 512 B coalesced read (4 strided u32 loads per lane);
//   * leaf blocks hold FL = 32 / 64 / 128 entries of S (u32) read together with
//     the matching col entries, so the pick's vertex arrives with the leaf;
//   * one 16 B record per vertex {leaf position, degree, index offset, T} is the
//     only per-vertex lookup (built when all four fit u32);
//   * leaves (S and a copy of col) are laid out 16 B aligned per row, and every
//     node starts 16 B aligned, so a group of G lanes can read a node with
//     uint4 loads: with G = 8 one warp walks 4 walkers at once.
// The searched values are the same integer prefix S_{i+1} = sum of deg over the
// first i+1 neighbours, so a pick is the same region s (Eq. 1) as
// the scan path and the oracle: bit-identical.
//
// Layout of row v (d = deg, rb = row start):
//   leaf     c32p[p + i] = S_{i+1} (u32), colp[p + i] = col[rb + i], i in [0, d),
//            p = leaf_pos(rb, v)
//   level k  (k >= 1) n_k = ceil(d / (FL * 128^(k-1))) entries; entry j = last S
//            of its child block; rows with d <= FL have no internal level.
//   K        = number of internal levels = first k with n_k <= 128 (top node);
//            stored top level first (each level padded to 4 entries) at inn[ioff[v] ...],
//            ioff = exclusive prefix of index_size over the vertices.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace csaw {

constexpr int WIX_NODE = 128;   // internal fanout
constexpr int WIX_NODE_LOG = 7;
// Vertex heads: one 512 B block per vertex at v * 512 B (address computable from v), words
// {d, T, leaf position, index offset} then 124 entries: the row's top index level when it
// has <= 124 entries, or, for rows of d <= 60, the whole leaf inline (S in words 4..63, col
// in words 64..123).  A step then starts with one coalesced read that carries the record
// and the first search level together (one dependent round trip less than record + node).
#ifndef WIX_HEAD_WORDS_N
#define WIX_HEAD_WORDS_N 128
#endif
constexpr int WIX_HEAD_WORDS = WIX_HEAD_WORDS_N;                 // 128 (512 B) or 256 (1 KB)
constexpr uint32_t WIX_HEAD_TOP = WIX_HEAD_WORDS - 4;             // inline top-level entries
constexpr uint32_t WIX_HEAD_LEAF = (WIX_HEAD_WORDS - 8) / 2;      // inline leaf entries (S and col)
constexpr int WIX_HEAD_NQ = WIX_HEAD_WORDS / 128;                 // uint4 per lane

template <int FL>
struct WixShape {
    static constexpr int kLeafLog = FL == 32 ? 5 : FL == 64 ? 6 : 7;
    // internal levels of a row of degree d
    __host__ __device__ __forceinline__ static int levels(uint32_t d) {
        if (d <= static_cast<uint32_t>(FL)) return 0;
        const int bits = 32 - clz32(d - 1);
        return (bits - kLeafLog + WIX_NODE_LOG - 1) / WIX_NODE_LOG;
    }
    // entries at level k >= 1
    __host__ __device__ __forceinline__ static uint32_t count(uint32_t d, int k) {
        return ((d - 1) >> (kLeafLog + WIX_NODE_LOG * (k - 1))) + 1;
    }
    __host__ __device__ __forceinline__ static uint32_t round4(uint32_t n) { return (n + 3) & ~3u; }
    // a row's index segment: its levels top first, each padded to a multiple of 4 entries
    // so every node starts 16 B aligned
    __host__ __device__ __forceinline__ static uint64_t index_size(uint32_t d) {
        uint64_t s = 0;
        const int K = levels(d);
        for (int k = 1; k <= K; ++k) s += round4(count(d, k));
        return s;
    }
    // start of row v's leaf entries in the padded leaf arrays (16 B aligned):
    // 4 ceil((rb + 3v) / 4); the gap to row v+1 is >= d.
    __host__ __device__ __forceinline__ static uint64_t leaf_pos(uint64_t rb, uint64_t v) {
        return (rb + 3 * v + 3) & ~uint64_t(3);
    }
    __host__ __device__ __forceinline__ static uint64_t leaf_total(uint64_t E, uint64_t V) {
        return E + 3 * V + 16;
    }
    __host__ __device__ __forceinline__ static int clz32(uint32_t x) {
#ifdef __CUDA_ARCH__
        return __clz(x);
#else
        return x ? __builtin_clz(x) : 32;
#endif
    }
};

// Entries base[q * 32 + lane], q < N, of one node / leaf block; entries past cnt read as
// 0xFFFFFFFF, which is above every draw (x < T <= 2^32 - 1).
template <int N>
__device__ __forceinline__ void wix_load(const uint32_t* __restrict__ p, uint32_t cnt, uint32_t (&v)[N]) {
    const uint32_t lane = static_cast<uint32_t>(lane_id());
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = q * 32 + lane < cnt ? __ldg(p + q * 32 + lane) : 0xFFFFFFFFu;
}
template <int N>
__device__ __forceinline__ uint32_t wix_pick(const uint32_t (&v)[N], uint32_t q) {
    uint32_t r = v[0];
#pragma unroll
    for (int i = 1; i < N; ++i) if (q == static_cast<uint32_t>(i)) r = v[i];
    return r;
}
// entry i of the block (all lanes)
template <int N>
__device__ __forceinline__ uint32_t wix_entry(const uint32_t (&v)[N], uint32_t i) {
    return __shfl_sync(FULL, wix_pick(v, i >> 5), i & 31);
}
// number of entries <= x = position of the first entry > x (the block is sorted)
template <int N>
__device__ __forceinline__ uint32_t wix_rank(const uint32_t (&v)[N], uint32_t x) {
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < N; ++q) c += v[q] <= x ? 1u : 0u;
    return __reduce_add_sync(FULL, c);
}

// uint4 component c (0..3) of q, c warp-uniform or per lane
__device__ __forceinline__ uint32_t u4_at(const uint4& q, uint32_t c) {
    return c == 0 ? q.x : c == 1 ? q.y : c == 2 ? q.z : q.w;
}


// Warp-collective search of row v for the draw x (< T): the region s with S_s <= x <
// S_{s+1}, through the vertex head (record + top level, or the inline row), the
// remaining internal nodes and one leaf.  Returns s, S_s (lo), b_s = S_{s+1} - S_s and
// col[s] -- what a without-replacement selection needs (BRS works on lo and b) -- and the
// bytes the search read.
template <int FL>
__device__ __forceinline__ void wix_head_search(const uint32_t* __restrict__ head, const uint32_t* __restrict__ c32p,
                                                const uint32_t* __restrict__ colp, const uint32_t* __restrict__ inn,
                                                uint32_t v, uint32_t x, uint32_t& s, uint32_t& lo, uint32_t& b,
                                                uint32_t& item, uint32_t& nbytes) {
    static_assert(WIX_HEAD_NQ == 1, "512 B heads");
    using W = WixShape<FL>;
    constexpr int NL = FL / 32;
    const uint32_t lane = static_cast<uint32_t>(lane_id());
    const uint4* hp = reinterpret_cast<const uint4*>(head + static_cast<uint64_t>(v) * WIX_HEAD_WORDS);
    const uint4 q = __ldg(hp + lane), hd = __ldg(hp);
    const uint32_t d = hd.x, p = hd.z, io = hd.w;
    auto head_entry = [&](uint32_t e) { return __shfl_sync(FULL, u4_at(q, e & 3), 1 + (e >> 2)); };
    auto head_rank = [&](uint32_t n) {
        uint32_t c = 0;
        if (lane >= 1) {
            const uint32_t e0 = 4 * (lane - 1);
            c = (e0 < n && q.x <= x) + (e0 + 1 < n && q.y <= x) + (e0 + 2 < n && q.z <= x) + (e0 + 3 < n && q.w <= x);
        }
        return __reduce_add_sync(FULL, c);
    };
    const int K = W::levels(d);
    nbytes = 4 * WIX_HEAD_WORDS;
    if (K == 0 && d <= WIX_HEAD_LEAF) {
        const uint32_t r = head_rank(d);
        const uint32_t hi = head_entry(r);
        lo = head_entry(r > 0 ? r - 1 : 0);
        if (r == 0) lo = 0;
        b = hi - lo;
        item = head_entry(WIX_HEAD_LEAF + r);
        s = r;
        return;
    }
    uint32_t j = 0, left = 0;
    uint64_t off = io;
    int k = K;
    if (K > 0) {
        const uint32_t nK = W::count(d, K);
        if (nK <= WIX_HEAD_TOP) {
            const uint32_t r = head_rank(nK);
            const uint32_t lv = head_entry(r > 0 ? r - 1 : 0);
            if (r > 0) left = lv;
            j = r;
            off += W::round4(nK);
            --k;
        }
    }
    for (; k >= 1; --k) {
        const uint32_t nk = W::count(d, k);
        const uint32_t cnt = min(static_cast<uint32_t>(WIX_NODE), nk - j * WIX_NODE);
        uint32_t vv[WIX_NODE / 32];
        wix_load(inn + off + static_cast<uint64_t>(j) * WIX_NODE, cnt, vv);
        nbytes += 4 * cnt;
        const uint32_t r = wix_rank(vv, x);
        const uint32_t lv = wix_entry(vv, r > 0 ? r - 1 : 0);
        if (r > 0) left = lv;
        j = j * WIX_NODE + r;
        off += W::round4(nk);
    }
    const uint64_t lb = static_cast<uint64_t>(p) + static_cast<uint64_t>(j) * FL;
    const uint32_t cnt = min(static_cast<uint32_t>(FL), d - j * FL);
    uint32_t sv[NL], cv[NL];
    wix_load(c32p + lb, cnt, sv);
    wix_load(colp + lb, cnt, cv);
    nbytes += 8 * cnt;
    const uint32_t r = wix_rank(sv, x);
    const uint32_t hi = wix_entry(sv, r);
    const uint32_t lv = wix_entry(sv, r > 0 ? r - 1 : 0);
    lo = r > 0 ? lv : left;
    b = hi - lo;
    item = wix_entry(cv, r);
    s = j * FL + r;
}

}  // namespace csaw
