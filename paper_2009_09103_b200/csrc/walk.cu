// walk.cu — random-walk kernels (with replacement): biased DeepWalk
// (degree), simple walk (uniform), node2vec and
// multi-dimensional random walk (Fig. 4).
//
// One warp owns one walker for its whole walk: the step loop runs inside the
// kernel (persistent; no host round trip per step).  Each step is
// one Select over N(cur) (§4.1): bias evaluation + Kogge-Stone CTPS in shared
// memory, one Philox draw keyed (instance, step), inverse transform search.
// Path entries are buffered one per lane and flushed as coalesced 128 B stores.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "internal.h"
#include "select.cuh"
#include "wix.cuh"

namespace csaw {

constexpr int WALK_WARPS = 8;   // warps per block

struct WalkArgs {
    const int64_t* __restrict__ rp;
    const uint32_t* __restrict__ col;
    const uint32_t* __restrict__ deg;
    const uint32_t* __restrict__ seeds;
    uint64_t n;
    int32_t L;
    uint32_t base;
    uint2 key;
    uint32_t* __restrict__ path;
    unsigned long long* __restrict__ counters;   // [0] = neighbours scanned, [1] = steps
    const uint64_t* __restrict__ ccache;          // chunk-total cache (degree pools), optional
};

// a9: warps fetch walkers from a global ticket (counters[7], zeroed per call),
// so warps whose walkers sit on hubs do not hold up the end of the launch.
__device__ __forceinline__ uint64_t walker_ticket(unsigned long long* ticket) {
    unsigned long long t = 0;
    if (lane_id() == 0) t = atomicAdd(ticket, 1ull);
    return __shfl_sync(FULL, t, 0);
}

// path[w][pi] buffered in lane (pi & 31); flushed when a 32-block completes.
struct PathWriter {
    uint32_t* row;
    uint32_t buf;
    int32_t L;
    __device__ __forceinline__ void put(int32_t pi, uint32_t v) {
        const int lane = lane_id();
        if ((pi & 31) == lane) buf = v;
        if ((pi & 31) == 31 || pi == L) {
            const int32_t idx = (pi & ~31) + lane;
            if (idx <= pi) row[idx] = buf;
        }
    }
};

// Degree-biased walk over the static-bias CTPS cache (NEXT-1): per step one row_ptr
// pair, one cache load for T, a 32-ary warp search of the cached prefix, one col
// load -- O(log32 d) round trips instead of an 8 d-byte rescan.  Bit-identical.
__global__ void __launch_bounds__(WALK_WARPS * 32, 4) k_walk_cached(WalkArgs a, const uint64_t* __restrict__ cps,
                                                                  const uint64_t* __restrict__ bt,
                                                                  const uint64_t* __restrict__ bt_off,
                                                                  const uint64_t* __restrict__ nmp) {
    const int lane = lane_id();
    unsigned long long probes = 0, steps = 0;
    for (uint64_t w = walker_ticket(a.counters + 7); w < a.n; w = walker_ticket(a.counters + 7)) {
        uint32_t cur = a.seeds[w];
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        PathWriter pw{a.path + w * (static_cast<uint64_t>(a.L) + 1), NONE, a.L};
        pw.put(0, cur);
        // current vertex's row: from row_ptr for the seed, then carried in nmp
        uint64_t rb = static_cast<uint64_t>(__ldg(a.rp + cur));
        uint32_t d = static_cast<uint32_t>(__ldg(a.rp + cur + 1) - static_cast<int64_t>(rb));
        uint64_t boff = __ldg(bt_off + cur);
        for (int32_t t = 0; t < a.L; ++t) {
            uint32_t nxt = NONE;
            if (cur != NONE && d > 0) {
                const uint64_t U = draw_u64(a.key, inst, static_cast<uint32_t>(t), 0u, word3(PURPOSE_EDGE, 0, 0));
                // B-tree over the cached prefix: T from the top level, one coalesced block
                // per level; col and the next vertex's (row, degree) read with the last block
                CpsTree tr{cps, bt, a.col, rb, d, boff};
                uint64_t x = 0, T = 0, e = 0, lo = 0, hi = 0, meta = 0;
                uint32_t pr = 0;
                if (nmp) {
                    tr.template search<true, true>(U, x, T, e, lo, hi, nxt, pr, nmp, &meta);
                    rb = meta >> 24;
                    d = static_cast<uint32_t>(meta & 0xFFFFFFu);
                    if (nxt != NONE) boff = __ldg(bt_off + nxt);
                } else {
                    tr.template search<true>(U, x, T, e, lo, hi, nxt, pr);
                    if (nxt != NONE) {
                        rb = static_cast<uint64_t>(__ldg(a.rp + nxt));
                        d = static_cast<uint32_t>(__ldg(a.rp + nxt + 1) - static_cast<int64_t>(rb));
                        boff = __ldg(bt_off + nxt);
                    }
                }
                probes += pr;
                if (T > 0) ++steps;
            }
            cur = nxt;
            pw.put(t + 1, cur);
        }
    }
    if (lane == 0) {
        if (probes) atomicAdd(a.counters + 2, probes);
        if (steps) atomicAdd(a.counters + 1, steps);
    }
}

// ---------------------------------------------------------------- narrow walk index (wix.cuh)
// Degree-biased walk over the narrow index, one warp per walker: per step one 16 B
// vertex record (with T, so the draw x is ready before the first node arrives), K <= 4 internal 512 B nodes (K = 0 for d <= FL, 1 for d <= 128 FL) and
// one leaf block with its col entries (4 strided u32 loads per lane and node).  The
// step's Philox draws are computed 32 at a time (lane j: step t0 + j) and broadcast, so
// the 10-round generator costs 1/32 per step.  Same S, same draws, same region as
// k_walk<degree> and the oracle (bit-identical).
template <int FL>
__global__ void __launch_bounds__(WALK_WARPS * 32, 4) k_walk_wix(WalkArgs a, const uint4* __restrict__ rec,
                                                               const uint32_t* __restrict__ c32p,
                                                               const uint32_t* __restrict__ colp,
                                                               const uint32_t* __restrict__ inn) {
    using W = WixShape<FL>;
    constexpr int NL = FL / 32;
    const int lane = lane_id();
    unsigned long long bytes = 0, steps = 0;
    for (uint64_t w = walker_ticket(a.counters + 7); w < a.n; w = walker_ticket(a.counters + 7)) {
        uint32_t cur = a.seeds[w];
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        PathWriter pw{a.path + w * (static_cast<uint64_t>(a.L) + 1), NONE, a.L};
        pw.put(0, cur);
        uint4 r = __ldg(rec + cur);   // {leaf position, degree, index offset, row total T}
        bytes += 16;
        uint64_t ubuf = 0;
        for (int32_t t = 0; t < a.L; ++t) {
            if ((t & 31) == 0)
                ubuf = draw_u64(a.key, inst, static_cast<uint32_t>(t + lane), 0u, word3(PURPOSE_EDGE, 0, 0));
            const uint64_t U = __shfl_sync(FULL, ubuf, t & 31);
            uint32_t nxt = NONE;
            const uint32_t d = r.y;
            if (cur != NONE && d > 0 && r.w > 0) {   // T = 0: no positive-bias neighbour, the walk ends (R20)
                const uint32_t x = static_cast<uint32_t>(below(U, r.w));
                const int K = W::levels(d);
                uint32_t j = 0;
                uint64_t off = r.z;
                for (int k = K; k >= 1; --k) {
                    const uint32_t nk = W::count(d, k);
                    const uint32_t cnt = min(static_cast<uint32_t>(WIX_NODE), nk - j * WIX_NODE);
                    uint32_t v[WIX_NODE / 32];
                    wix_load(inn + off + j * WIX_NODE, cnt, v);
                    bytes += 4ull * cnt;
                    j = j * WIX_NODE + wix_rank(v, x);
                    off += W::round4(nk);
                }
                const uint64_t lb = static_cast<uint64_t>(r.x) + static_cast<uint64_t>(j) * FL;
                const uint32_t cnt = min(static_cast<uint32_t>(FL), d - j * FL);
                uint32_t v[NL], cv[NL];
                wix_load(c32p + lb, cnt, v);
                wix_load(colp + lb, cnt, cv);
                bytes += 8ull * cnt;
                nxt = wix_entry(cv, wix_rank(v, x));
                ++steps;
            }
            cur = nxt;
            pw.put(t + 1, cur);
            if (cur != NONE) {
                r = __ldg(rec + cur);
                bytes += 16;
            }
        }
    }
    if (lane == 0) {
        if (bytes) atomicAdd(a.counters + 3, bytes);
        if (steps) atomicAdd(a.counters + 1, steps);
    }
}

#ifndef GB_WARPS
#define GB_WARPS 2
#endif
// Degree-biased walk over the bucketed index (CSAW_GRAPH_WALK_BUCKETS, capi.cu build_gb): a step
// is x = below(U, T), ONE 128 B line -- bucket x >> k of the current vertex, 8 entries read by
// lanes 0..7 -- and the last entry with S_i <= x, which carries the next vertex with its own
// bucket table, shift and T: one dependent DRAM round trip per step (k_walk_head: head, then
// leaf).  A link entry (a bucket met by more than 8 regions, ~0.2 % of cfg2's steps) continues
// in the row's CTPS cache 32 entries at a time, then reads the pick's col and bucket metadata.
// Same S, same draw, same region as every other degree-walk kernel and the oracle.
__global__ void __launch_bounds__(WALK_WARPS * 32, 4) k_walk_gb(WalkArgs a, const uint4* __restrict__ gbk,
                                                              const uint4* __restrict__ gmeta,
                                                              const uint64_t* __restrict__ cps, uint64_t E,
                                                              uint64_t nbk) {
    const int lane = lane_id();
    unsigned long long bytes = 0, steps = 0, links = 0;
    for (uint64_t w = walker_ticket(a.counters + 7); w < a.n; w = walker_ticket(a.counters + 7)) {
        uint32_t cur = a.seeds[w];
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        PathWriter pw{a.path + w * (static_cast<uint64_t>(a.L) + 1), NONE, a.L};
        pw.put(0, cur);
        const uint4 m0 = __ldg(gmeta + cur);
        uint32_t B = m0.x, k = m0.y, T = m0.z;
        uint64_t ubuf = 0;
        for (int32_t t = 0; t < a.L; ++t) {
            if ((t & 31) == 0)
                ubuf = draw_u64(a.key, inst, static_cast<uint32_t>(t + lane), 0u, word3(PURPOSE_EDGE, 0, 0));
            const uint64_t U = __shfl_sync(FULL, ubuf, t & 31);
            uint32_t nxt = NONE;
            if (cur != NONE && T > 0) {   // T = 0: no positive-bias neighbour, the walk ends (R20)
                const uint32_t x = static_cast<uint32_t>(below(U, T));
                uint4 e = make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);
                CSAW_DASSERT(static_cast<uint64_t>(B) + (x >> k) < nbk);
                if (lane < 8) e = __ldg(gbk + (static_cast<uint64_t>(B) + (x >> k)) * 8 + lane);
                const int fl = 31 - __clz(__ballot_sync(FULL, lane < 8 && e.x <= x));   // entry 0 always passes
                const uint32_t uk = __shfl_sync(FULL, e.y, fl);
                const uint32_t eb = __shfl_sync(FULL, e.z, fl), et = __shfl_sync(FULL, e.w, fl);
                bytes += 128;
                if (uk != 0xFFFFFFFFu) {
                    nxt = uk & 0x7FFFFFFu;
                    k = uk >> 27;
                    B = eb;
                    T = et;
                } else {   // link: the region of x lies at or after CSR entry ge of this row
                    ++links;
                    uint64_t ge = static_cast<uint64_t>(et) << 32 | eb;
                    for (;;) {   // first entry with inclusive prefix > x (exists: x < T)
                        const uint64_t c = ge + lane < E ? __ldg(cps + ge + lane) : ~0ull;
                        const unsigned gt = __ballot_sync(FULL, c > x);
                        bytes += 256;
                        if (gt) { ge += __ffs(gt) - 1; break; }
                        ge += 32;
                    }
                    CSAW_DASSERT(ge < E);
                    nxt = __ldg(a.col + ge);
                    const uint4 mu = __ldg(gmeta + nxt);
                    B = mu.x;
                    k = mu.y;
                    T = mu.z;
                    bytes += 20;
                }
                ++steps;
            }
            cur = nxt;
            pw.put(t + 1, nxt);
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (bytes) atomicAdd(a.counters + 3, bytes + 4ull * steps);
        if (steps) atomicAdd(a.counters + 1, steps);
        if (links) atomicAdd(a.counters + 2, links);
    }
}

// Edge-weight walk (float path, R28) over the weighted bucketed index (capi.cu build_gbw): x =
// r(U) T in fp64, bucket floor(x 2^-k), one 128 B line of 5 SoA entries read by lanes 0..4, the
// last entry with S <= x -- it carries the next vertex, its bucket table, shift and fp64 T.  The
// row sums are the oracle's left-to-right fp64 sums, so every pick is the oracle's (no boundary
// excuse).  A link entry continues in the row's fp64 prefix: the last positive-weight region
// with S_excl <= x, 32 entries at a time.
__global__ void __launch_bounds__(WALK_WARPS * 32, 4) k_walk_gbw(WalkArgs a, const uint8_t* __restrict__ gbw,
                                                               const uint4* __restrict__ meta,
                                                               const double* __restrict__ cpsw,
                                                               const float* __restrict__ w, uint64_t nbk) {
    constexpr int CAP = 5, KB = 24;
    const int lane = lane_id();
    unsigned long long bytes = 0, steps = 0, links = 0;
    for (uint64_t wk = walker_ticket(a.counters + 7); wk < a.n; wk = walker_ticket(a.counters + 7)) {
        uint32_t cur = a.seeds[wk];
        const uint32_t inst = a.base + static_cast<uint32_t>(wk);
        PathWriter pw{a.path + wk * (static_cast<uint64_t>(a.L) + 1), NONE, a.L};
        pw.put(0, cur);
        const uint4 m0 = __ldg(meta + cur);
        uint32_t B = m0.x;
        int k = static_cast<int>(m0.y) - KB;
        double T = __longlong_as_double(static_cast<long long>(static_cast<uint64_t>(m0.w) << 32 | m0.z));
        uint64_t ubuf = 0;
        for (int32_t t = 0; t < a.L; ++t) {
            if ((t & 31) == 0)
                ubuf = draw_u64(a.key, inst, static_cast<uint32_t>(t + lane), 0u, word3(PURPOSE_EDGE, 0, 0));
            const uint64_t U = __shfl_sync(FULL, ubuf, t & 31);
            uint32_t nxt = NONE;
            if (cur != NONE && T > 0.0) {   // T = 0: every weight of the row is 0, the walk ends (R20)
                const double x = (static_cast<double>(U >> 11) * (1.0 / 9007199254740992.0)) * T;
                const uint64_t bi = static_cast<uint64_t>(ldexp(x, -k));
                CSAW_DASSERT(static_cast<uint64_t>(B) + bi < nbk);
                const uint8_t* line = gbw + (static_cast<uint64_t>(B) + bi) * 128;
                double S = __longlong_as_double(0x7FF0000000000000ll), Tu = 0.0;
                uint32_t uk = 0, Bu = 0;
                if (lane < CAP) {
                    S = __ldg(reinterpret_cast<const double*>(line) + lane);
                    Tu = __ldg(reinterpret_cast<const double*>(line) + CAP + lane);
                    uk = __ldg(reinterpret_cast<const uint32_t*>(line + 16 * CAP) + lane);
                    Bu = __ldg(reinterpret_cast<const uint32_t*>(line + 20 * CAP) + lane);
                }
                const int fl = 31 - __clz(__ballot_sync(FULL, lane < CAP && S <= x));   // entry 0 always passes
                const uint32_t uks = __shfl_sync(FULL, uk, fl);
                const double Ts = __shfl_sync(FULL, Tu, fl);
                const uint32_t Bs = __shfl_sync(FULL, Bu, fl);
                bytes += 128;
                if (uks != 0xFFFFFFFFu) {
                    nxt = uks & 0x7FFFFFFu;
                    k = static_cast<int>(uks >> 27) - KB;
                    B = Bs;
                    T = Ts;
                } else {   // link: the last positive region with S_excl <= x at or after CSR entry j0
                    ++links;
                    uint64_t j0 = static_cast<uint64_t>(__double_as_longlong(Ts));
                    const uint64_t re = static_cast<uint64_t>(__ldg(a.rp + cur + 1));
                    uint64_t best = j0;   // entry j0 itself qualifies (S_excl(j0) <= x, positive)
                    for (;; j0 += 32) {
                        const uint64_t j = j0 + lane;
                        const bool in = j < re;
                        const double sxj = in ? __ldg(cpsw + j - 1) : __longlong_as_double(0x7FF0000000000000ll);
                        const bool le = sxj <= x;
                        const unsigned ok = __ballot_sync(FULL, le && in && __ldg(w + j) > 0.0f);
                        if (ok) best = j0 + (31 - __clz(ok));
                        bytes += 384;
                        if (!__shfl_sync(FULL, le, 31)) break;   // a later entry starts beyond x (or the row ended)
                    }
                    nxt = __ldg(a.col + best);
                    const uint4 mu = __ldg(meta + nxt);
                    B = mu.x;
                    k = static_cast<int>(mu.y) - KB;
                    T = __longlong_as_double(static_cast<long long>(static_cast<uint64_t>(mu.w) << 32 | mu.z));
                    bytes += 20;
                }
                ++steps;
            }
            cur = nxt;
            pw.put(t + 1, nxt);
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (bytes) atomicAdd(a.counters + 3, bytes + 4ull * steps);
        if (steps) atomicAdd(a.counters + 1, steps);
        if (links) atomicAdd(a.counters + 2, links);
    }
}

// Degree-biased walk over the vertex heads (wix.cuh): a step is one coalesced 512 B head
// read (record + top level, or the whole row when d <= 60), then K - 1 internal nodes and
// one leaf when the row is larger -- one dependent round trip less than record + nodes.
// Same S, same draws, same region as k_walk_wix / k_walk<degree> / the oracle.
template <int FL>
__global__ void __launch_bounds__(WALK_WARPS * 32, 4) k_walk_head(WalkArgs a, const uint32_t* __restrict__ head,
                                                                const uint32_t* __restrict__ c32p,
                                                                const uint32_t* __restrict__ colp,
                                                                const uint32_t* __restrict__ inn) {
    using W = WixShape<FL>;
    constexpr int NL = FL / 32;
    const uint32_t lane = static_cast<uint32_t>(lane_id());
    unsigned long long bytes = 0, steps = 0;
    for (uint64_t w = walker_ticket(a.counters + 7); w < a.n; w = walker_ticket(a.counters + 7)) {
        uint32_t cur = a.seeds[w];
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        PathWriter pw{a.path + w * (static_cast<uint64_t>(a.L) + 1), NONE, a.L};
        pw.put(0, cur);
        uint64_t ubuf = 0;
        // the head of the vertex a step starts from is requested as soon as that vertex is
        // known (end of the previous step); every lane also loads the 16 B header itself
        // (same line, one transaction), so no shuffles sit between the head and the draw
        constexpr int NQ = WIX_HEAD_NQ;   // lane l holds head words 4 NQ l .. 4 NQ l + 4 NQ - 1
        const uint4* hp = reinterpret_cast<const uint4*>(head + static_cast<uint64_t>(cur) * WIX_HEAD_WORDS);
        uint4 q[NQ];
#pragma unroll
        for (int i = 0; i < NQ; ++i) q[i] = __ldg(hp + NQ * lane + i);
        uint4 hd = __ldg(hp);
        for (int32_t t = 0; t < a.L; ++t) {
            if ((t & 31) == 0)
                ubuf = draw_u64(a.key, inst, static_cast<uint32_t>(t + lane), 0u, word3(PURPOSE_EDGE, 0, 0));
            const uint64_t U = __shfl_sync(FULL, ubuf, t & 31);
            uint32_t nxt = NONE;
            if (cur != NONE) {
                const uint32_t d = hd.x, T = hd.y, p = hd.z, io = hd.w;
                bytes += 4 * WIX_HEAD_WORDS;
                if (d > 0 && T > 0) {   // T = 0: no positive-bias neighbour, the walk ends (R20)
                    const uint32_t x = static_cast<uint32_t>(below(U, T));
                    const int K = W::levels(d);
                    // rank of x among the head's entries [0, n): entry e is word 4 + e
                    auto head_rank = [&](uint32_t n) {
                        uint32_t c = 0;
#pragma unroll
                        for (int i = 0; i < NQ; ++i) {
                            const uint32_t w0 = 4 * (NQ * lane + i);   // first word of q[i]
                            if (w0 >= 4) {
                                const uint32_t e0 = w0 - 4;
                                c += (e0 < n && q[i].x <= x) + (e0 + 1 < n && q[i].y <= x) +
                                     (e0 + 2 < n && q[i].z <= x) + (e0 + 3 < n && q[i].w <= x);
                            }
                        }
                        return __reduce_add_sync(FULL, c);
                    };
                    if (K == 0 && d <= WIX_HEAD_LEAF) {   // the whole row is in the head
                        const uint32_t r = head_rank(d);
                        const uint32_t wc = 4 + WIX_HEAD_LEAF + r;   // col entry r
                        const uint32_t qi = (wc >> 2) % NQ;
                        uint4 qq = q[0];
#pragma unroll
                        for (int i = 1; i < NQ; ++i) if (qi == static_cast<uint32_t>(i)) qq = q[i];
                        nxt = __shfl_sync(FULL, u4_at(qq, wc & 3), wc / (4 * NQ));
                    } else {
                        uint32_t j = 0;
                        uint64_t off = io;
                        int k = K;
                        if (K > 0) {
                            const uint32_t nK = W::count(d, K);
                            if (nK <= WIX_HEAD_TOP) {   // top level inline
                                j = head_rank(nK);
                                off += W::round4(nK);
                                --k;
                            }
                        }
                        for (; k >= 1; --k) {
                            const uint32_t nk = W::count(d, k);
                            const uint32_t cnt = min(static_cast<uint32_t>(WIX_NODE), nk - j * WIX_NODE);
                            uint32_t v[WIX_NODE / 32];
                            wix_load(inn + off + j * WIX_NODE, cnt, v);
                            bytes += 4ull * cnt;
                            j = j * WIX_NODE + wix_rank(v, x);
                            off += W::round4(nk);
                        }
                        const uint64_t lb = static_cast<uint64_t>(p) + static_cast<uint64_t>(j) * FL;
                        const uint32_t cnt = min(static_cast<uint32_t>(FL), d - j * FL);
                        uint32_t v[NL], cv[NL];
                        wix_load(c32p + lb, cnt, v);
                        wix_load(colp + lb, cnt, cv);
                        bytes += 8ull * cnt;
                        nxt = wix_entry(cv, wix_rank(v, x));
                    }
                    ++steps;
                }
            }
            cur = nxt;
            if (cur != NONE && t + 1 < a.L) {
                const uint4* np = reinterpret_cast<const uint4*>(head + static_cast<uint64_t>(cur) * WIX_HEAD_WORDS);
#pragma unroll
                for (int i = 0; i < NQ; ++i) q[i] = __ldg(np + NQ * lane + i);
                hd = __ldg(np);
            }
            pw.put(t + 1, cur);
        }
    }
    if (lane == 0) {
        if (bytes) atomicAdd(a.counters + 3, bytes);
        if (steps) atomicAdd(a.counters + 1, steps);
    }
}

// One node / leaf block read by a group of G lanes: lane gl holds entries 4 gl + 4 G i .. +3
// (i < N), 16 B aligned uint4 loads; entries past cnt read as 0xFFFFFFFF (above every draw).
template <int G, int N>
__device__ __forceinline__ void wixg_load(const uint32_t* __restrict__ p, uint32_t cnt, int gl, uint4 (&q)[N]) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const uint32_t e0 = 4 * gl + 4 * G * i;
        q[i] = e0 < cnt ? __ldg(reinterpret_cast<const uint4*>(p + e0)) : make_uint4(~0u, ~0u, ~0u, ~0u);
        if (e0 + 1 >= cnt) q[i].y = ~0u;
        if (e0 + 2 >= cnt) q[i].z = ~0u;
        if (e0 + 3 >= cnt) q[i].w = ~0u;
    }
}
template <int N>
__device__ __forceinline__ uint32_t wixg_count(const uint4 (&q)[N], uint32_t x) {
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) c += (q[i].x <= x) + (q[i].y <= x) + (q[i].z <= x) + (q[i].w <= x);
    return c;
}

// Sub-warp variant: G lanes per walker, 32/G walkers per warp.  The chain of dependent
// loads per step is the same (record -> K nodes -> leaf), but one warp instruction now
// advances 32/G walkers, so the SM issue slots per walker step drop ~32/G-fold (the
// warp-per-walker kernel was ~50 % issue-bound at cfg2), at the price of lockstep: each
// step waits for the slowest of the warp's walkers.  Draws: lane gl computes step t0 + gl
// every G steps.  Bit-identical to k_walk_wix.
template <int G, int FL>
__global__ void __launch_bounds__(WALK_WARPS * 32, 4) k_walk_wixg(WalkArgs a, const uint4* __restrict__ rec,
                                                                const uint32_t* __restrict__ c32p,
                                                                const uint32_t* __restrict__ colp,
                                                                const uint32_t* __restrict__ inn) {
    using W = WixShape<FL>;
    constexpr int NI = WIX_NODE / (4 * G);   // uint4 chunks per lane: internal node
    constexpr int NF = FL / (4 * G);         // uint4 chunks per lane: leaf block
    static_assert(NF >= 1 && NI >= 1, "FL must be a multiple of 4 G");
    const int lane = lane_id();
    const int gl = lane % G;
    const int gb = lane - gl;
    const uint64_t ngroups = total_warps() * (32 / G);
    const uint64_t gid0 = global_warp_id() * (32 / G) + static_cast<uint64_t>(lane / G);
    const uint64_t rounds = (a.n + ngroups - 1) / ngroups;   // warp-uniform trip count (shuffles below)
    unsigned long long bytes = 0, steps = 0;
    for (uint64_t rd = 0; rd < rounds; ++rd) {
        const uint64_t w = gid0 + rd * ngroups;
        const bool live = w < a.n;
        uint32_t cur = live ? a.seeds[w] : NONE;
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        uint32_t* prow = a.path + (live ? w : 0) * (static_cast<uint64_t>(a.L) + 1);
        uint32_t pbuf = cur;                  // path[pi] buffered in lane pi % G
        uint4 r = make_uint4(0, 0, 0, 0);
        if (cur != NONE) {
            r = __ldg(rec + cur);
            if (gl == 0) bytes += 16;
        }
        if (live && a.L == 0 && gl == 0) prow[0] = pbuf;
        uint64_t ubuf = 0;
        for (int32_t t = 0; t < a.L; ++t) {
            if (t % G == 0)
                ubuf = draw_u64(a.key, inst, static_cast<uint32_t>(t + gl), 0u, word3(PURPOSE_EDGE, 0, 0));
            const uint64_t U = __shfl_sync(FULL, ubuf, gb + t % G);
            const uint32_t d = r.y;
            const bool on = cur != NONE && d > 0 && r.w > 0;   // T = 0: the walk ends (R20)
            const uint32_t x = static_cast<uint32_t>(below(U, r.w));
            const int K = on ? W::levels(d) : 0;
            const int Kmax = static_cast<int>(__reduce_max_sync(FULL, static_cast<uint32_t>(K)));
            uint32_t j = 0;
            uint64_t off = r.z;
            for (int k = Kmax; k >= 1; --k) {
                const bool act = on && k <= K;
                uint32_t c = 0;
                if (act) {
                    const uint32_t nk = W::count(d, k);
                    const uint32_t cnt = min(static_cast<uint32_t>(WIX_NODE), nk - j * WIX_NODE);
                    uint4 q[NI];
                    wixg_load<G>(inn + off + j * WIX_NODE, cnt, gl, q);
                    if (gl == 0) bytes += 4ull * cnt;
                    c = wixg_count(q, x);
                    off += W::round4(nk);
                }
#pragma unroll
                for (int o = G / 2; o >= 1; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
                if (act) j = j * WIX_NODE + c;
            }
            uint32_t c = 0;
            uint4 cv[NF];
            if (on) {
                const uint64_t lb = static_cast<uint64_t>(r.x) + static_cast<uint64_t>(j) * FL;
                const uint32_t cnt = min(static_cast<uint32_t>(FL), d - j * FL);
                uint4 q[NF];
                wixg_load<G>(c32p + lb, cnt, gl, q);
#pragma unroll
                for (int i = 0; i < NF; ++i) {
                    const uint32_t e0 = 4 * gl + 4 * G * i;
                    cv[i] = e0 < cnt ? __ldg(reinterpret_cast<const uint4*>(colp + lb + e0)) : make_uint4(0, 0, 0, 0);
                }
                if (gl == 0) bytes += 8ull * cnt;
                c = wixg_count(q, x);
            } else {
#pragma unroll
                for (int i = 0; i < NF; ++i) cv[i] = make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int o = G / 2; o >= 1; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
            // entry c of the leaf: chunk c / (4 G), lane (c / 4) % G of the group, component c % 4
            uint32_t val = 0;
            const uint32_t ci = c / (4 * G), cc = c & 3;
#pragma unroll
            for (int i = 0; i < NF; ++i)
                if (ci == static_cast<uint32_t>(i)) val = cc == 0 ? cv[i].x : cc == 1 ? cv[i].y : cc == 2 ? cv[i].z : cv[i].w;
            val = __shfl_sync(FULL, val, gb + static_cast<int>((c >> 2) % G));
            uint32_t nxt = NONE;
            if (on) {
                nxt = val;
                if (gl == 0) ++steps;
            }
            cur = nxt;
            // path[t + 1]: buffered in lane (t + 1) % G, flushed as one G x 4 B segment
            const int32_t pi = t + 1;
            if (pi % G == gl) pbuf = cur;
            if (live && (pi % G == G - 1 || pi == a.L)) {
                const int32_t idx = pi - pi % G + gl;
                if (idx <= pi) prow[idx] = pbuf;
            }
            if (cur != NONE) {
                r = __ldg(rec + cur);
                if (gl == 0) bytes += 16;
            }
        }
    }
    if (gl == 0) {
        if (bytes) atomicAdd(a.counters + 3, bytes);
        if (steps) atomicAdd(a.counters + 1, steps);
    }
}

template <bool kUniform>
__global__ void __launch_bounds__(WALK_WARPS * 32) k_walk(WalkArgs a) {
    __shared__ uint64_t tab_all[WALK_WARPS][TAB];
    uint64_t* tab = tab_all[threadIdx.x >> 5];
    const int lane = lane_id();
    unsigned long long scanned = 0, steps = 0;
    for (uint64_t w = walker_ticket(a.counters + 7); w < a.n; w = walker_ticket(a.counters + 7)) {
        uint32_t cur = a.seeds[w];
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        PathWriter pw{a.path + w * (static_cast<uint64_t>(a.L) + 1), NONE, a.L};
        pw.put(0, cur);
        for (int32_t t = 0; t < a.L; ++t) {
            uint32_t nxt = NONE;
            if (cur != NONE) {
                const int64_t b0 = __ldg(a.rp + cur);
                const uint32_t d = static_cast<uint32_t>(__ldg(a.rp + cur + 1) - b0);
                if (d > 0) {
                    const uint64_t U = draw_u64(a.key, inst, static_cast<uint32_t>(t), 0u, word3(PURPOSE_EDGE, 0, 0));
                    if constexpr (kUniform) {
                        nxt = __ldg(a.col + b0 + below(U, d));
                    } else {
                        DegreePool P{a.col, a.deg, static_cast<uint64_t>(b0), d, a.ccache};
                        const Ctps C = build_ctps(P, tab);
                        nxt = select_wr(P, C, tab, U);
                        scanned += (a.ccache && C.m) ? 32u * C.m : d;   // chunk cache: one chunk rescanned
                    }
                    ++steps;
                }
            }
            cur = nxt;
            pw.put(t + 1, cur);
        }
    }
    if (lane == 0) {
        if (scanned) atomicAdd(a.counters + 0, scanned);
        if (steps) atomicAdd(a.counters + 1, steps);
    }
}

// ---------------------------------------------------------------- Table-1 walk variants (NEXT-3)
// Metropolis-Hastings, restart and jump walks:
// a uniform proposal u = N(v)[below(U(EDGE), d)] plus one extra keyed draw.
template <int kKind>   // CSAW_BIAS_MH / RESTART / JUMP
__global__ void __launch_bounds__(WALK_WARPS * 32) k_walk_variant(WalkArgs a, uint64_t theta, int64_t V) {
    const int lane = lane_id();
    unsigned long long steps = 0;
    for (uint64_t w = walker_ticket(a.counters + 7); w < a.n; w = walker_ticket(a.counters + 7)) {
        const uint32_t s0 = a.seeds[w];
        uint32_t cur = s0;
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        PathWriter pw{a.path + w * (static_cast<uint64_t>(a.L) + 1), NONE, a.L};
        pw.put(0, cur);
        for (int32_t t = 0; t < a.L; ++t) {
            uint32_t nxt = NONE;
            const uint32_t tt = static_cast<uint32_t>(t);
            if (cur != NONE) {
                bool jumped = false;
                if constexpr (kKind == CSAW_BIAS_RESTART || kKind == CSAW_BIAS_JUMP) {
                    const uint4 o = philox4x32_10(make_uint4(inst, tt, 0u, word3(PURPOSE_JUMP, 0, 0)), a.key);
                    if (static_cast<uint64_t>(o.x) < theta) {
                        jumped = true;
                        if constexpr (kKind == CSAW_BIAS_RESTART) nxt = s0;
                        else nxt = static_cast<uint32_t>(below(draw_u64(a.key, inst, tt, 0u, word3(PURPOSE_TARGET, 0, 0)),
                                                               static_cast<uint64_t>(V)));
                    }
                }
                if (!jumped) {
                    const int64_t b0 = __ldg(a.rp + cur);
                    const uint32_t d = static_cast<uint32_t>(__ldg(a.rp + cur + 1) - b0);
                    if (d > 0) {
                        const uint32_t u = __ldg(a.col + b0 + below(draw_u64(a.key, inst, tt, 0u, word3(PURPOSE_EDGE, 0, 0)), d));
                        nxt = u;
                        if constexpr (kKind == CSAW_BIAS_MH) {
                            const uint32_t du = __ldg(a.deg + u);
                            const uint64_t acc = below(draw_u64(a.key, inst, tt, 0u, word3(PURPOSE_ACCEPT, 0, 0)), du);
                            if (!(acc < d)) nxt = cur;   // rejected: stay
                        }
                    }
                }
                ++steps;
            }
            cur = nxt;
            pw.put(t + 1, cur);
        }
    }
    if (lane == 0 && steps) atomicAdd(a.counters + 1, steps);
}

// ---------------------------------------------------------------- node2vec
// EdgeBias of u in N(v) with predecessor prev: class 0 (u == prev, alpha 1/p),
// class 1 (u in N(prev), alpha 1), class 2 (otherwise, alpha 1/q) -- Grover &
// Leskovec's second-order bias (reading R16).  Membership in the
// sorted N(prev) is a warp-cooperative merge: rows of N(v) (ascending) are
// matched against a 32-entry window of N(prev) held one per lane, searched
// with 5 shuffle steps; the window only moves forward (32-ary jumps).
struct Node2vecPool {
    static constexpr bool kClosedForm = false;
    static constexpr bool kCached = false;
    const uint32_t* __restrict__ col;
    uint64_t beg;       // N(v) = col[beg, beg + n)
    uint32_t n;
    const uint32_t* __restrict__ nprev;   // N(prev) = nprev[0, np)
    uint64_t np;
    uint32_t prev;
    uint32_t w[3];      // bias per class (integer path), or class codes {0,1,2} (float path)
    // merge state
    uint64_t wp;        // window start in N(prev)
    uint32_t W;         // lane's window element (NONE beyond np)
    bool wvalid;

    __device__ __forceinline__ void seek(uint32_t) { wvalid = false; wp = 0; }

    __device__ __forceinline__ void load_window(uint64_t at) {
        wp = at;
        const uint64_t p = at + lane_id();
        W = p < np ? __ldg(nprev + p) : NONE;
        wvalid = true;
    }

    // Move the window forward so that it contains lower_bound(N(prev), key): first
    // the adjacent window (one coalesced load; the common case when merging lists
    // of similar size), else a 32-ary search of the remainder.
    __device__ __forceinline__ void advance_to(uint32_t key) {
        if (!wvalid) {
            load_window(warp_lower_bound(nprev, 0, np, key));
            return;
        }
        if (wp + 32 >= np) {   // window already covers the tail
            load_window(np);
            return;
        }
        load_window(wp + 32);
        if (__shfl_sync(FULL, W, 31) < key && wp + 32 < np) load_window(warp_lower_bound(nprev, wp + 32, np, key));
    }

    // membership of each lane's u (ascending across lanes; NONE = invalid lane)
    __device__ __forceinline__ bool member_row(uint32_t u) {
        const bool valid = u != NONE;
        const unsigned vm = __ballot_sync(FULL, valid);
        if (!vm || np == 0) return false;
        const uint32_t umin = __shfl_sync(FULL, u, __ffs(vm) - 1);
        if (!wvalid || __shfl_sync(FULL, W, 31) < umin) advance_to(umin);
        bool mem = false, open = valid;
        for (;;) {
            // lower_bound of u in the 32-entry window by shuffle binary search
            int idx = 0;
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                const uint32_t wv = __shfl_sync(FULL, W, idx + s - 1);
                if (wv < u) idx += s;
            }
            const bool found = __shfl_sync(FULL, W, idx) == u;
            const uint32_t w31 = __shfl_sync(FULL, W, 31);
            if (open && u <= w31) { mem = found; open = false; }
            const unsigned om = __ballot_sync(FULL, open);
            if (!om) break;
            const uint32_t un = __shfl_sync(FULL, u, __ffs(om) - 1);
            advance_to(un);
        }
        return mem;
    }

    template <int NR>
    __device__ __forceinline__ void load_rows(uint32_t row0, uint32_t (&key)[NR], uint32_t (&b)[NR]) {
        const int lane = lane_id();
#pragma unroll
        for (int u = 0; u < NR; ++u) {
            const uint32_t i = (row0 + u) * 32 + lane;
            key[u] = (i < n) ? __ldg(col + beg + i) : NONE;
        }
#pragma unroll
        for (int u = 0; u < NR; ++u) {
            const bool mem = member_row(key[u]);
            b[u] = key[u] == NONE ? 0u : (key[u] == prev ? w[0] : (mem ? w[1] : w[2]));
        }
    }
    __device__ __forceinline__ uint32_t item(uint32_t i) const { return __ldg(col + beg + i); }
};

struct N2vArgs {
    WalkArgs wa;
    uint32_t wint[3];    // integer biases {m/p, m, m/q} (R16); unused on the float path
    float wf[3];         // float biases {(float)(1/p), 1, (float)(1/q)}
    const float* __restrict__ ew = nullptr;   // edge weights: b = alpha * w(e) (R33), float path
};

// Float CTPS (general p, q): fp32 biases summed in fp64 (north star; R28).
__device__ __forceinline__ double warp_incl_scan_f64(double v) {
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// The float bias of pool entry i: alpha (class code c) times the edge weight when weighted.
__device__ __forceinline__ double n2v_fbias(const Node2vecPool& P, const float (&wf)[3], const float* __restrict__ ew,
                                            bool first, uint32_t key, uint32_t c, uint32_t i) {
    if (key == NONE) return 0.0;
    const float a = first ? 1.0f : wf[c];
    if (!ew) return static_cast<double>(a);
    return static_cast<double>(__fmul_rn(a, __ldg(ew + P.beg + i)));   // one fp32 multiply (R33)
}

// One float-path step: x = r*T with r = (U >> 11) 2^-53; s = first i with b_i > 0 and
// S_{i+1} > x (past every boundary through rounding: the last positive entry).  Two passes:
// totals per chunk of U rows, then a rescan.  ew (nullable): b_i = fp32(alpha_i * w_i) (R33);
// first: the weighted step 0 (b_i = w_i).
__device__ uint32_t n2v_float_step(Node2vecPool& P, const float (&wf)[3], double* ftab, uint64_t U64,
                                   const float* __restrict__ ew = nullptr, bool first = false) {
    const int lane = lane_id();
    const uint32_t n = P.n;
    const uint32_t nrows = (n + 31) >> 5;
    const uint32_t m = max(static_cast<uint32_t>(U), ((nrows + TAB - 1) / TAB + U - 1) / U * U);
    double carry = 0.0;
    uint32_t chunk = 0;
    P.seek(0);
    for (uint32_t c0 = 0; c0 < nrows; c0 += m) {
        const uint32_t c1 = min(c0 + m, nrows);
        for (uint32_t r0 = c0; r0 < c1; r0 += U) {
            uint32_t key[U], b[U];
            P.template load_rows<U>(r0, key, b);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double bv = n2v_fbias(P, wf, ew, first, key[u], b[u], (r0 + u) * 32 + lane);
                carry += __shfl_sync(FULL, warp_incl_scan_f64(bv), 31);
            }
        }
        if (lane == 0) ftab[chunk] = carry;
        ++chunk;
    }
    __syncwarp();
    const double T = carry;
    const double r = static_cast<double>(U64 >> 11) * (1.0 / 9007199254740992.0);
    const double x = r * T;
    uint32_t c = 0;
    while (c + 1 < chunk && ftab[c] <= x) ++c;   // chunk containing x (clamped to the last)
    double base = c ? ftab[c - 1] : 0.0;
    const uint32_t rbeg = c * m;
    P.seek(rbeg);
    uint32_t last_item = NONE;
    for (uint32_t r0 = rbeg; r0 < nrows; r0 += U) {   // past the chunk only through rounding
        uint32_t key[U], b[U];
        P.template load_rows<U>(r0, key, b);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double bv = n2v_fbias(P, wf, ew, first, key[u], b[u], (r0 + u) * 32 + lane);
            const double incl = warp_incl_scan_f64(bv) + base;
            const unsigned hit = __ballot_sync(FULL, bv > 0.0 && incl > x);
            const unsigned vm = __ballot_sync(FULL, bv > 0.0);
            if (vm) last_item = __shfl_sync(FULL, key[u], 31 - __clz(vm));
            if (hit) return __shfl_sync(FULL, key[u], __ffs(hit) - 1);
            base = __shfl_sync(FULL, incl, 31);
        }
    }
    return last_item;   // x >= T after rounding: the last positive candidate
}

// Integer node2vec step with an implicit CTPS.  The bias of u in N(v) takes only
// three values -- w[0] (u == prev), w[1] (u in N(prev)), w[2] (otherwise) -- so
// S_i = w2 * (#regular before i) + sum of the special weights before i.  One merge
// pass over N(v) x N(prev) records the "special" positions (prev and the common
// neighbours) in shared memory; T and the region of x follow in closed form
// between consecutive specials.  Same integers as the scanned CTPS, so the same
// pick.  Returns false if more than SPEC_CAP specials (caller uses the scan).
constexpr uint32_t SPEC_CAP = 1024;

// Membership of each lane's x (ascending over valid lanes) in big[lo0, nb), by
// narrowing: [lo, hi) = the big-list range of the row's value span (two 32-ary
// searches), then one shuffle search if it fits a window, else a per-lane binary
// search.  lo0 advances monotonically (rows are processed in ascending order).
__device__ __forceinline__ bool n2v_find(const uint32_t* __restrict__ big, uint64_t& lo0, uint64_t nb, uint32_t x,
                                         bool valid, uint64_t& idx) {
    const int lane = lane_id();
    const unsigned vm = __ballot_sync(FULL, valid);
    idx = 0;
    if (!vm || lo0 >= nb) return false;
    const uint32_t xmin = __shfl_sync(FULL, x, __ffs(vm) - 1);
    const uint32_t xmax = __shfl_sync(FULL, x, 31 - __clz(vm));
    const uint64_t lo = warp_lower_bound(big, lo0, nb, xmin);
    const uint64_t hi = warp_lower_bound(big, lo, nb, xmax + 1u);
    lo0 = hi;
    bool found = false;
    if (hi - lo <= 32) {
        const uint32_t W = (lo + lane < hi) ? __ldg(big + lo + lane) : NONE;
        int k = 0;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            const uint32_t wv = __shfl_sync(FULL, W, k + s - 1);
            if (wv < x) k += s;
        }
        const uint32_t wk = __shfl_sync(FULL, W, k);   // all lanes shuffle (no short-circuit)
        found = valid && wk == x;
        idx = lo + k;
    } else {
        uint64_t l = lo, h = hi;
        while (l < h) {   // same trip count on every lane (same range)
            const uint64_t mid = (l + h) >> 1;
            if (__ldg(big + mid) < x) l = mid + 1; else h = mid;
        }
        found = valid && l < hi && __ldg(big + l) == x;
        idx = l;
    }
    return found;
}

constexpr uint32_t TILE_N = 512;   // N(prev) tile (u32) in shared memory (reuses the CTPS table)

// Enumerates the special positions of N(v) -- prev and the common neighbours with
// N(prev) -- in ascending order; stores those of rank [skip, skip + SPEC_CAP) in
// spec[rank - skip] (bit 31 = prev).  Returns the total count.
__device__ uint32_t n2v_specials(Node2vecPool& P, uint32_t* spec, uint32_t* tilebuf, uint32_t skip, bool& has_prev) {
    const int lane = lane_id();
    const uint32_t n = P.n;
    const uint32_t nrows = (n + 31) >> 5;
    uint32_t cnt = 0;
    has_prev = false;
    const uint64_t dv = n, dp = P.np;
    if (dp <= 8 * dv && dv <= 8 * dp) {
        // balanced sizes: merge 8-row chunks of N(v) (registers) against 512-entry
        // tiles of N(prev) staged in shared memory -- coalesced loads, each list read
        // once, membership by a branch-free binary search in the tile
        uint32_t* tile = tilebuf;
        uint64_t bpos = 0;
        uint32_t tn = 0, tmax = 0;
        auto load_tile = [&](uint64_t at) {
            bpos = at;
            tn = static_cast<uint32_t>(min(static_cast<uint64_t>(TILE_N), dp - at));
            __syncwarp();
            for (uint32_t j = lane; j < tn; j += 32) tile[j] = __ldg(P.nprev + at + j);
            __syncwarp();
            tmax = tile[tn - 1];
        };
        load_tile(0);
        for (uint32_t r0 = 0; r0 < nrows; r0 += U) {
            uint32_t key[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = (r0 + u) * 32 + lane;
                key[u] = (i < n) ? __ldg(P.col + P.beg + i) : NONE;
            }
            uint32_t open = 0, memmask = 0;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (key[u] != NONE && key[u] != P.prev) open |= 1u << u;
            for (;;) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (((open >> u) & 1u) && key[u] <= tmax) {
                        uint32_t pos = 0;
#pragma unroll
                        for (uint32_t st = TILE_N / 2; st > 0; st >>= 1)
                            if (pos + st <= tn && tile[pos + st - 1] < key[u]) pos += st;
                        if (pos < tn && tile[pos] == key[u]) memmask |= 1u << u;
                        open &= ~(1u << u);
                    }
                }
                if (!__any_sync(FULL, open != 0)) break;
                if (bpos + tn >= dp) break;            // N(prev) exhausted: the rest are not members
                load_tile(bpos + tn);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (r0 + u < nrows) {
                    const bool isp = key[u] == P.prev;
                    const bool sp = key[u] != NONE && (isp || ((memmask >> u) & 1u));
                    const unsigned bal = __ballot_sync(FULL, sp);
                    if (sp) {
                        const uint32_t idx = cnt + __popc(bal & lanemask_lt());
                        if (idx >= skip && idx - skip < SPEC_CAP) spec[idx - skip] = ((r0 + u) * 32 + lane) | (isp ? 0x80000000u : 0u);
                    }
                    has_prev |= __any_sync(FULL, isp);
                    cnt += __popc(bal);
                }
            }
        }
    } else {
        // imbalanced: iterate the smaller list, narrowed search in the larger one
        const uint32_t* A = P.col + P.beg;    // N(v)
        const uint64_t pp = warp_lower_bound(A, 0, dv, P.prev);
        has_prev = pp < dv && __ldg(A + pp) == P.prev;
        const bool small_is_v = dv < dp;
        const uint32_t* small = small_is_v ? A : P.nprev;
        const uint32_t* big = small_is_v ? P.nprev : A;
        const uint64_t ns = small_is_v ? dv : dp, nb = small_is_v ? dp : dv;
        uint64_t lo0 = 0;
        bool prev_done = !has_prev;
        for (uint64_t r0 = 0; r0 < ns; r0 += 32) {
            const uint64_t i = r0 + lane;
            const bool valid = i < ns;
            const uint32_t xv = valid ? __ldg(small + i) : NONE;
            uint64_t bi = 0;
            const bool f = n2v_find(big, lo0, nb, xv, valid, bi);
            const bool mem = f && xv != P.prev;
            const uint64_t posA = small_is_v ? i : bi;      // position in N(v)
            // insert prev's own position in order (it is not in N(prev): no self-loops)
            if (!prev_done) {
                const unsigned before = __ballot_sync(FULL, mem && posA < pp);
                const unsigned after = __ballot_sync(FULL, mem && posA > pp);
                (void)before;
                if (after || r0 + 32 >= ns) {
                    // emit members < pp first, then prev, then the rest of this row
                    const unsigned bal0 = __ballot_sync(FULL, mem && posA < pp);
                    if (mem && posA < pp) {
                        const uint32_t idx = cnt + __popc(bal0 & lanemask_lt());
                        if (idx >= skip && idx - skip < SPEC_CAP) spec[idx - skip] = static_cast<uint32_t>(posA);
                    }
                    cnt += __popc(bal0);
                    if (lane == 0 && cnt >= skip && cnt - skip < SPEC_CAP) spec[cnt - skip] = static_cast<uint32_t>(pp) | 0x80000000u;
                    ++cnt;
                    prev_done = true;
                    const unsigned bal1 = __ballot_sync(FULL, mem && posA > pp);
                    if (mem && posA > pp) {
                        const uint32_t idx = cnt + __popc(bal1 & lanemask_lt());
                        if (idx >= skip && idx - skip < SPEC_CAP) spec[idx - skip] = static_cast<uint32_t>(posA);
                    }
                    cnt += __popc(bal1);
                    continue;
                }
            }
            const unsigned bal = __ballot_sync(FULL, mem);
            if (mem) {
                const uint32_t idx = cnt + __popc(bal & lanemask_lt());
                if (idx >= skip && idx - skip < SPEC_CAP) spec[idx - skip] = static_cast<uint32_t>(posA);
            }
            cnt += __popc(bal);
        }
        if (!prev_done) {   // empty small list
            if (lane == 0 && cnt >= skip && cnt - skip < SPEC_CAP) spec[cnt - skip] = static_cast<uint32_t>(pp) | 0x80000000u;
            ++cnt;
        }
    }
    __syncwarp();
    return cnt;
}

// Integer node2vec step with an implicit CTPS (see above).  Specials beyond the
// shared-memory window are handled by re-enumerating the next window.
__device__ void n2v_implicit_step(Node2vecPool& P, uint32_t* spec, uint32_t* tilebuf, uint64_t U64, uint32_t& out) {
    const int lane = lane_id();
    const uint32_t n = P.n;
    const uint64_t wp = P.w[0], w1 = P.w[1], wq = P.w[2];
    bool has_prev = false;
    const uint32_t cnt = n2v_specials(P, spec, tilebuf, 0, has_prev);
    const uint64_t np_ = has_prev ? 1 : 0;
    const uint64_t T = wq * (n - cnt) + w1 * (cnt - np_) + wp * np_;
    const uint64_t x = below(U64, T);
    // largest special j with S(p_j) = wq * (p_j - j) + sum_{j' < j} w_j' <= x
    bool found = false, stop = false;
    uint64_t Ssel = 0, wsel = 0, psel = 0, base = 0;
    for (uint32_t win = 0; win < cnt && !stop; win += SPEC_CAP) {
        if (win > 0) {
            bool hp;
            n2v_specials(P, spec, tilebuf, win, hp);
        }
        const uint32_t wn = min(SPEC_CAP, cnt - win);
        for (uint32_t j0 = 0; j0 < wn; j0 += 32) {
            const uint32_t jl = j0 + lane;
            const uint64_t j = win + jl;
            const bool valid = jl < wn;
            const uint32_t e = valid ? spec[jl] : 0u;
            const uint64_t pos = e & 0x7FFFFFFFu;
            const uint64_t wj = valid ? ((e >> 31) ? wp : w1) : 0;
            const uint64_t incl = warp_incl_scan(wj);
            const uint64_t Sj = wq * (pos - j) + base + incl - wj;
            const unsigned vm = __ballot_sync(FULL, valid);
            const unsigned le = __ballot_sync(FULL, valid && Sj <= x);
            if (le) {
                const int f = 31 - __clz(le);
                found = true;
                Ssel = __shfl_sync(FULL, Sj, f);
                wsel = __shfl_sync(FULL, wj, f);
                psel = __shfl_sync(FULL, pos, f);
            }
            if (le != vm) { stop = true; break; }
            base += __shfl_sync(FULL, incl, 31);
        }
        __syncwarp();
    }
    uint64_t i;
    if (!found) i = x / wq;
    else if (x < Ssel + wsel) i = psel;
    else i = psel + 1 + (x - Ssel - wsel) / wq;
    out = __ldg(P.col + P.beg + i);
}

// ---------------------------------------------------------------- node2vec with edge triangle counts
// With tri[e] = |N(v) ∩ N(prev)| (capi.cu build_tri; symmetric graphs) the step's row total
// is closed-form: T = wq (d - C - 1) + w1 C + wp (prev is in N(v), C common neighbours).
// The draw x then fixes the region without a full merge: N(v) is scanned from the end
// nearer to x (x < T/2: forward; else backward, as a forward scan of the mirrored lists
// with x' = T - 1 - x -- bitwise NOT reverses u32 order, so both directions share one
// code path) only until the running S passes x.  Expected scan length: a quarter of
// N(v) instead of all of it plus all of N(prev).  Same S, same x, same region as the
// scanned CTPS and the oracle (bit-identical).
#ifndef N2T_TILE_N
#define N2T_TILE_N 1024
#endif
constexpr uint32_t N2T_TILE = N2T_TILE_N;   // N(prev) window in shared memory (u32), per warp
#ifndef N2T_KEYS
#define N2T_KEYS 4
#endif
constexpr int N2T_K = N2T_KEYS;
#ifndef N2T_BS_RATIO
#define N2T_BS_RATIO 4u      // N(prev) this much longer than N(v): per-key binary searches of N(prev) (cfg3: 4x 714, 8x 715, 16x 727, 64x 774 ms)
#endif
#ifndef N2T_SPEC_RATIO
#define N2T_SPEC_RATIO 8u   // N(prev) this much shorter than N(v): specials by search, no scan of N(v) (cfg3: 2x 777, 4x 727, 8x 727, 16x 750 ms)
#endif       // keys per lane per chunk (contiguous positions)
constexpr int N2T_WARPS = 8;
#ifndef N2T_MINB
#define N2T_MINB 4   // 64 registers, 32 warps / SM: the step is latency-bound (cfg3: 3: 714, 4: 543, 5: 699 (spills), 6: 972 ms)
#endif

// A sorted list read forwards, or backwards with every value complemented (x -> ~x
// reverses u32 order, so the mirrored list is ascending too): at(i) = p[b + s i] ^ m with
// (b, s, m) = (0, 1, 0) or (n - 1, -1, ~0).  One code path for both scan directions (a
// template per direction doubled the kernel and stalled on instruction fetch).
struct MirList {
    const uint32_t* __restrict__ p;   // p[0] = the first element in scan order
    uint32_t n;
    int32_t s;                         // +1 / -1
    uint32_t m;                        // 0 / 0xFFFFFFFF
    __device__ __forceinline__ uint32_t at(uint32_t i) const {
        return __ldg(p + static_cast<int64_t>(s) * static_cast<int64_t>(i)) ^ m;
    }
};
__device__ __forceinline__ MirList mir_list(const uint32_t* p, uint32_t n, bool rev) {
    return rev ? MirList{p + (n ? n - 1 : 0), n, -1, 0xFFFFFFFFu} : MirList{p, n, 1, 0u};
}

// First idx in [lo, hi) with L.at(idx) >= key (hi if none); 32-ary warp search.
__device__ __forceinline__ uint32_t mir_lower_bound(const MirList& L, uint32_t lo, uint32_t hi, uint32_t key) {
    const uint32_t lane = static_cast<uint32_t>(lane_id());
    while (hi - lo > 32) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t p = lo + lane * step;
        const bool inr = p < hi;
        const unsigned b = __ballot_sync(FULL, inr && L.at(p) >= key);
        const unsigned inb = __ballot_sync(FULL, inr);
        if (b == 0) {
            lo = lo + static_cast<uint32_t>(31 - __clz(inb)) * step + 1;
        } else {
            const uint32_t f = static_cast<uint32_t>(__ffs(b) - 1);
            if (f == 0) return lo;
            const uint32_t nlo = lo + (f - 1) * step + 1;
            hi = lo + f * step;
            lo = nlo;
        }
    }
    const uint32_t p = lo + lane;
    const unsigned b = __ballot_sync(FULL, p < hi && L.at(p) >= key);
    return b ? lo + static_cast<uint32_t>(__ffs(b) - 1) : hi;
}

struct N2tStats {
    unsigned long long keys = 0;    // N(v) entries scanned
    unsigned long long bkeys = 0;   // N(prev) entries read (tiles / searches)
};

// Position (in A's order) of the region containing xs: first i with S_{i+1} > xs, where
// S sums w(A[j]) = wp (A[j] == pvk), w1 (A[j] in B), wq (otherwise).  Chunks of 256 keys,
// lane l holding the 8 consecutive positions 8 l .. 8 l + 7; membership against a
// shared-memory tile of B: per lane one binary search for its first key, then a linear
// merge (B about as dense as A) or galloping searches (B denser); B much longer than A:
// per-key binary searches of B in global memory.
// Splitters: every step-th entry of a (mirrored) list staged in shared memory with
// cp.async (one round trip), so a key's lower bound is narrowed to a window of `step`
// entries by a shared-memory search before the global binary search (log2(step) round
// trips instead of log2(n)).
#ifndef N2T_SPLIT
#define N2T_SPLIT 256u    // splitters staged per list (<= N2T_TILE; cfg3: 1024: 480, 256: 476, 128: 482 ms)
#endif
struct Splitters {
    uint32_t ns, step;
};
__device__ __forceinline__ Splitters stage_splitters(const MirList& L, uint32_t* tile) {
    const uint32_t lane = static_cast<uint32_t>(lane_id());
    Splitters sp;
    sp.step = max(1u, (L.n + N2T_SPLIT - 1) / N2T_SPLIT);
    sp.ns = (L.n + sp.step - 1) / sp.step;
    __syncwarp();
    for (uint32_t i = lane; i < sp.ns; i += 32) {
        const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(tile + i));
        const uint32_t* src = L.p + static_cast<int64_t>(L.s) * static_cast<int64_t>(i * sp.step);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    if (L.m)
        for (uint32_t i = lane; i < sp.ns; i += 32) tile[i] ^= L.m;
    __syncwarp();
    return sp;
}
// [l, h): the lower bound of k in L lies in [l, h] (h when every entry of [l, h) is < k)
__device__ __forceinline__ void split_window(const uint32_t* tile, const Splitters& sp, uint32_t n, uint32_t k,
                                             uint32_t& l, uint32_t& h) {
    uint32_t c = 0;   // splitters < k, in [0, ns] (ns <= N2T_TILE: the first step may take all of them)
#pragma unroll
    for (uint32_t s = N2T_TILE; s > 0; s >>= 1)
        if (c + s <= sp.ns && tile[c + s - 1] < k) c += s;
    if (c == 0) { l = 0; h = 0; return; }   // L[0] >= k
    l = (c - 1) * sp.step + 1;
    h = c < sp.ns ? c * sp.step : n;
}

// B much shorter than A (N(prev) << N(v)): instead of scanning A, locate the specials --
// B's members of A (weight w1) and prev (weight wp) -- by searching each B entry in A;
// between specials S grows by wq per position, so the region follows in closed form.
// S(p) at a member at position p with j members before it: wq p - (wq - w1) j -
// (wq - wp) [p > ppos].  Members come in ascending position (B is sorted), so the walk
// over B stops at the first member whose S passes xs.
__device__ uint32_t n2t_specials(const MirList& A, const MirList& B, uint32_t pvk, uint64_t xs, uint32_t wp,
                                 uint32_t w1, uint32_t wq, uint32_t* tile, N2tStats& st) {
    const uint32_t lane = static_cast<uint32_t>(lane_id());
    const uint32_t ppos = mir_lower_bound(A, 0, A.n, pvk);   // prev is in N(v) (symmetric graph)
    const Splitters sp = stage_splitters(A, tile);
    // deficits per special (mod 2^64: negative when 1/q < 1 or 1/q < 1/p; S itself is exact)
    const uint64_t dq1 = static_cast<uint64_t>(wq) - w1, dqp = static_cast<uint64_t>(wq) - wp;
    uint32_t j = 0;                 // members seen so far
    uint32_t before_prev = 0;       // members at positions < ppos
    bool have = false;              // a member with S <= xs seen
    uint32_t pm = 0;                // its position (the last such)
    uint64_t Sm = 0;
    bool stop = false;
    for (uint32_t r0 = 0; r0 < B.n && !stop; r0 += 32) {
        const uint32_t i = r0 + lane;
        const bool valid = i < B.n;
        const uint32_t b = valid ? B.at(i) : 0u;
        uint32_t l = 0, h = 0;
        if (valid) split_window(tile, sp, A.n, b, l, h);
        for (uint32_t span = sp.step; span > 0; span >>= 1) {   // same trip count on every lane
            if (l < h) {
                const uint32_t mid = (l + h) >> 1;
                if (A.at(mid) < b) l = mid + 1; else h = mid;
            }
        }
        const bool mem = valid && l < A.n && A.at(l) == b;
        st.bkeys += min(32u, B.n - r0) * (32 - __clz(sp.step + 1));
        const unsigned mb = __ballot_sync(FULL, mem);
        const uint32_t jj = j + __popc(mb & lanemask_lt());   // members before this one
        const uint64_t S = static_cast<uint64_t>(wq) * l - dq1 * jj - (l > ppos ? dqp : 0);
        const unsigned le = __ballot_sync(FULL, mem && S <= xs);
        if (le) {
            const int f = 31 - __clz(le);
            have = true;
            pm = __shfl_sync(FULL, l, f);
            Sm = __shfl_sync(FULL, S, f);
        }
        before_prev += __popc(__ballot_sync(FULL, mem && l < ppos));
        if (__ballot_sync(FULL, mem && S > xs)) stop = true;   // later members only grow S
        j += __popc(mb);
    }
    // prev as a special: S(ppos) = wq ppos - (wq - w1) (members before it); complete if
    // the walk stopped after ppos (else S(ppos) > xs anyway, see above)
    const uint64_t Sp = static_cast<uint64_t>(wq) * ppos - dq1 * before_prev;
    uint32_t q;
    uint64_t Sq, wqq;
    if (Sp <= xs && (!have || ppos > pm)) { q = ppos; Sq = Sp; wqq = wp; }
    else if (have) { q = pm; Sq = Sm; wqq = w1; }
    else return static_cast<uint32_t>(xs / wq);   // before every special
    if (xs < Sq + wqq) return q;
    return q + 1 + static_cast<uint32_t>((xs - Sq - wqq) / wq);
}

__device__ uint32_t n2t_scan(const MirList& A, const MirList& B, uint32_t pvk, uint64_t xs, uint32_t wp,
                             uint32_t w1, uint32_t wq, uint32_t* tile, N2tStats& st) {
    const uint32_t lane = static_cast<uint32_t>(lane_id());
    if (N2T_SPEC_RATIO * B.n < A.n) return n2t_specials(A, B, pvk, xs, wp, w1, wq, tile, st);
    const bool bsearch = B.n > N2T_BS_RATIO * A.n;
    const bool linear = B.n <= 3u * A.n;
    uint64_t acc = 0;
    uint32_t bnext = 0;                     // B entries before bnext are below every key still to come
    uint32_t tlo = 0, tn = 0, tmax = 0;     // tile = B[tlo, tlo + tn)
    bool tile_ok = false;
    Splitters bsp{0, 1};                    // bsearch mode: splitters of B in the tile
    for (uint32_t c0 = 0; c0 < A.n; c0 += 32 * N2T_K) {
        const uint32_t base = c0 + N2T_K * lane;
        const uint32_t nv = base < A.n ? min(static_cast<uint32_t>(N2T_K), A.n - base) : 0u;   // valid keys of the lane
        uint32_t k[N2T_K];
#pragma unroll
        for (int u = 0; u < N2T_K; ++u) k[u] = static_cast<uint32_t>(u) < nv ? A.at(base + u) : 0u;
        const uint32_t cn = min(static_cast<uint32_t>(32 * N2T_K), A.n - c0);
        st.keys += cn;
        uint32_t mem = 0;
        if (bsearch) {
            if (c0 == 0) bsp = stage_splitters(B, tile);   // once per step (bnext stays 0 in this mode)
            uint32_t l[N2T_K], h[N2T_K];
#pragma unroll
            for (int u = 0; u < N2T_K; ++u) {
                l[u] = 0; h[u] = 0;
                if (static_cast<uint32_t>(u) < nv) split_window(tile, bsp, B.n, k[u], l[u], h[u]);
            }
            for (uint32_t span = bsp.step; span > 0; span >>= 1) {   // same trip count on all lanes
#pragma unroll
                for (int u = 0; u < N2T_K; ++u) {
                    if (l[u] < h[u]) {
                        const uint32_t mid = (l[u] + h[u]) >> 1;
                        if (B.at(mid) < k[u]) l[u] = mid + 1; else h[u] = mid;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < N2T_K; ++u)
                if (static_cast<uint32_t>(u) < nv && l[u] < B.n && B.at(l[u]) == k[u]) mem |= 1u << u;
            st.bkeys += static_cast<unsigned long long>(cn) * (32 - __clz(bsp.step + 1));
        } else if (bnext < B.n) {
            uint32_t open = 0;
#pragma unroll
            for (int u = 0; u < N2T_K; ++u)
                if (static_cast<uint32_t>(u) < nv && k[u] != pvk) open |= 1u << u;
            for (;;) {
                if (!tile_ok) {
                    tlo = bnext;
                    tn = min(N2T_TILE, B.n - bnext);
                    __syncwarp();
                    // global -> shared without a register round trip per element: all of the
                    // lane's copies are in flight at once (cp.async), then mirrored lists are
                    // complemented in place
                    for (uint32_t j = lane; j < tn; j += 32) {
                        const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(tile + j));
                        const uint32_t* src = B.p + static_cast<int64_t>(B.s) * static_cast<int64_t>(tlo + j);
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src) : "memory");
                    }
                    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
                    if (B.m)
                        for (uint32_t j = lane; j < tn; j += 32) tile[j] ^= B.m;
                    __syncwarp();
                    tmax = tile[tn - 1];
                    tile_ok = true;
                    st.bkeys += tn;
                }
                // the lane's open keys <= tmax: binary search for the first, then merge / gallop
                uint32_t first = N2T_K;
#pragma unroll
                for (int u = N2T_K - 1; u >= 0; --u)
                    if (((open >> u) & 1u) && k[u] <= tmax) first = u;
                if (first < N2T_K) {
                    uint32_t k0 = k[0];
#pragma unroll
                    for (int u = 1; u < N2T_K; ++u) if (first == static_cast<uint32_t>(u)) k0 = k[u];
                    uint32_t p = 0;
#pragma unroll
                    for (uint32_t s = N2T_TILE / 2; s > 0; s >>= 1)
                        if (p + s <= tn && tile[p + s - 1] < k0) p += s;
#pragma unroll
                    for (int u = 0; u < N2T_K; ++u) {
                        if (((open >> u) & 1u) && k[u] <= tmax) {
                            if (linear) {
                                while (p < tn && tile[p] < k[u]) ++p;
                            } else {
                                uint32_t step = 1;
                                while (p + step <= tn && tile[p + step - 1] < k[u]) { p += step; step <<= 1; }
                                uint32_t hi = min(p + step - 1, tn);
                                while (p < hi) {
                                    const uint32_t mid = (p + hi) >> 1;
                                    if (tile[mid] < k[u]) p = mid + 1; else hi = mid;
                                }
                            }
                            if (p < tn && tile[p] == k[u]) mem |= 1u << u;
                            open &= ~(1u << u);
                        }
                    }
                }
                if (!__any_sync(FULL, open != 0)) break;
                // smallest key still open (positions ascend with u, then lane)
                uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
                for (int u = N2T_K - 1; u >= 0; --u)
                    if ((open >> u) & 1u) kmin = k[u];
                kmin = __reduce_min_sync(FULL, kmin);
                bnext = tlo + tn;
                tile_ok = false;
                if (bnext >= B.n) break;   // B exhausted: the open keys are not members
                bnext = mir_lower_bound(B, bnext, B.n, kmin);
                if (bnext >= B.n) break;
            }
        }
        // running S: lane-local prefix of 8 weights, warp scan of the lane totals
        uint32_t loc[N2T_K];
        uint32_t tot = 0;
#pragma unroll
        for (int u = 0; u < N2T_K; ++u) {
            const uint32_t w = static_cast<uint32_t>(u) < nv ? (k[u] == pvk ? wp : ((mem >> u) & 1u) ? w1 : wq) : 0u;
            tot += w;
            loc[u] = tot;
        }
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        const uint64_t lbase = acc + (incl - tot);   // S before the lane's first key
        const unsigned hit = __ballot_sync(FULL, nv > 0 && lbase + tot > xs);
        if (hit) {
            const int f = __ffs(hit) - 1;
            uint32_t pos = 0;
            if (lane == static_cast<uint32_t>(f)) {
                pos = N2T_K - 1;
#pragma unroll
                for (int u = N2T_K - 1; u >= 0; --u)
                    if (lbase + loc[u] > xs) pos = u;
            }
            return c0 + N2T_K * f + __shfl_sync(FULL, pos, f);
        }
        acc += __shfl_sync(FULL, incl, 31);
    }
    return A.n - 1;   // not reached for xs < T
}

__global__ void __launch_bounds__(N2T_WARPS * 32, N2T_MINB) k_node2vec_tri(N2vArgs na, const uint32_t* __restrict__ tri) {
    __shared__ uint32_t tile_all[N2T_WARPS][N2T_TILE];
    uint32_t* tile = tile_all[threadIdx.x >> 5];
    const WalkArgs& a = na.wa;
    const uint32_t wp = na.wint[0], w1 = na.wint[1], wq = na.wint[2];
    const int lane = lane_id();
    N2tStats st;
    unsigned long long steps = 0;
    for (uint64_t w = walker_ticket(a.counters + 7); w < a.n; w = walker_ticket(a.counters + 7)) {
        uint32_t cur = a.seeds[w], prev = NONE;
        uint64_t e_in = 0;   // CSR entry prev -> cur
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        PathWriter pw{a.path + w * (static_cast<uint64_t>(a.L) + 1), NONE, a.L};
        pw.put(0, cur);
        uint64_t ubuf = 0;
        for (int32_t t = 0; t < a.L; ++t) {
            if ((t & 31) == 0)
                ubuf = draw_u64(a.key, inst, static_cast<uint32_t>(t + lane), 0u, word3(PURPOSE_EDGE, 0, 0));
            const uint64_t U = __shfl_sync(FULL, ubuf, t & 31);
            uint32_t nxt = NONE;
            if (cur != NONE) {
                const int64_t b0 = __ldg(a.rp + cur);
                const uint32_t d = static_cast<uint32_t>(__ldg(a.rp + cur + 1) - b0);
                if (d > 0) {
                    uint32_t s;
                    if (prev == NONE) {
                        s = static_cast<uint32_t>(below(U, d));   // step 0: uniform (R16)
                    } else {
                        const uint32_t C = __ldg(tri + e_in);
                        const uint64_t T = static_cast<uint64_t>(wq) * (d - C - 1) + static_cast<uint64_t>(w1) * C + wp;
                        const uint64_t x = below(U, T);
                        const int64_t p0 = __ldg(a.rp + prev);
                        const uint32_t dp = static_cast<uint32_t>(__ldg(a.rp + prev + 1) - p0);
                        const bool rev = 2 * x >= T;   // mirrored: the same forward scan from the end
                        const MirList A = mir_list(a.col + b0, d, rev), B = mir_list(a.col + p0, dp, rev);
                        const uint32_t sp = n2t_scan(A, B, rev ? ~prev : prev, rev ? T - 1 - x : x, wp, w1, wq, tile, st);
                        s = rev ? d - 1 - sp : sp;
                    }
                    e_in = static_cast<uint64_t>(b0) + s;
                    nxt = __ldg(a.col + e_in);
                    ++steps;
                }
            }
            prev = cur;
            cur = nxt;
            pw.put(t + 1, cur);
        }
    }
    if (lane == 0) {   // bytes: row_ptr pairs of v and prev, tri, the pick's col, + 4 per list entry read
        if (st.keys + st.bkeys) atomicAdd(a.counters + 0, st.keys + st.bkeys);
        if (steps) atomicAdd(a.counters + 1, steps);
        atomicAdd(a.counters + 3, 4ull * (st.keys + st.bkeys) + 40ull * steps);
    }
}

template <bool kFloat>
__global__ void __launch_bounds__(WALK_WARPS * 32, 3) k_node2vec(N2vArgs na) {
    __shared__ uint64_t tab_all[WALK_WARPS][TAB];
    __shared__ uint32_t spec_all[kFloat ? 1 : WALK_WARPS][kFloat ? 1 : SPEC_CAP];
    uint64_t* tab = tab_all[threadIdx.x >> 5];
    uint32_t* spec = spec_all[kFloat ? 0 : (threadIdx.x >> 5)];
    const WalkArgs& a = na.wa;
    const int lane = lane_id();
    unsigned long long scanned = 0, steps = 0;
    for (uint64_t w = walker_ticket(a.counters + 7); w < a.n; w = walker_ticket(a.counters + 7)) {
        uint32_t cur = a.seeds[w], prev = NONE;
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        PathWriter pw{a.path + w * (static_cast<uint64_t>(a.L) + 1), NONE, a.L};
        pw.put(0, cur);
        for (int32_t t = 0; t < a.L; ++t) {
            uint32_t nxt = NONE;
            if (cur != NONE) {
                const int64_t b0 = __ldg(a.rp + cur);
                const uint32_t d = static_cast<uint32_t>(__ldg(a.rp + cur + 1) - b0);
                if (d > 0) {
                    const uint64_t U64 = draw_u64(a.key, inst, static_cast<uint32_t>(t), 0u, word3(PURPOSE_EDGE, 0, 0));
                    if (prev == NONE && !(kFloat && na.ew)) {
                        nxt = __ldg(a.col + b0 + below(U64, d));     // step 0: uniform (R16)
                    } else if (prev == NONE) {                       // weighted step 0: b = w (R33)
                        Node2vecPool P;
                        P.col = a.col; P.beg = static_cast<uint64_t>(b0); P.n = d;
                        P.nprev = a.col; P.np = 0; P.prev = NONE;
                        P.wp = 0; P.W = NONE; P.wvalid = false;
                        P.w[0] = 0; P.w[1] = 1; P.w[2] = 2;
                        nxt = n2v_float_step(P, na.wf, reinterpret_cast<double*>(tab), U64, na.ew, true);
                        scanned += d;
                    } else {
                        const int64_t p0 = __ldg(a.rp + prev);
                        Node2vecPool P;
                        P.col = a.col; P.beg = static_cast<uint64_t>(b0); P.n = d;
                        P.nprev = a.col + p0;
                        P.np = static_cast<uint64_t>(__ldg(a.rp + prev + 1) - p0);
                        P.prev = prev;
                        P.wp = 0; P.W = NONE; P.wvalid = false;
                        if constexpr (kFloat) {
                            P.w[0] = 0; P.w[1] = 1; P.w[2] = 2;
                            nxt = n2v_float_step(P, na.wf, reinterpret_cast<double*>(tab), U64, na.ew);
                        } else {
                            P.w[0] = na.wint[0]; P.w[1] = na.wint[1]; P.w[2] = na.wint[2];
                            n2v_implicit_step(P, spec, reinterpret_cast<uint32_t*>(tab), U64, nxt);
                        }
                        scanned += d;
                    }
                    ++steps;
                }
            }
            prev = cur;
            cur = nxt;
            pw.put(t + 1, cur);
        }
    }
    if (lane == 0) {
        if (scanned) atomicAdd(a.counters + 0, scanned);
        if (steps) atomicAdd(a.counters + 1, steps);
    }
}

// Host twin of the oracle's reading R16 (independent code): smallest m in
// [1, 2^16] with m/p and m/q integers in [1, 2^32); 0 = float path.
static uint32_t n2v_integer_scale(double p, double q) {
    for (uint32_t m = 1; m <= 65536u; ++m) {
        const double a = static_cast<double>(m) / p, c = static_cast<double>(m) / q;
        if (a == std::floor(a) && c == std::floor(c) && a >= 1.0 && c >= 1.0 && a < 4294967296.0 && c < 4294967296.0)
            return m;
    }
    return 0;
}

// ---------------------------------------------------------------- MDRW
// Multi-dimensional random walk (frontier sampling; Fig. 4): per
// instance a pool of m vertices in slot order (R18).  VertexBias = degree:
// the warp keeps the m biases and per-32-slot block totals (shared memory),
// so a draw is located by a warp scan over block totals then one over a block
// -- exactly ITS over the slot-order CTPS.  EdgeBias = 1 (closed form, one col
// load), Update replaces the picked slot in place.
struct MdrwArgs {
    const int64_t* __restrict__ rp;
    const uint32_t* __restrict__ col;
    const uint32_t* __restrict__ seeds;   // [n][m]
    uint64_t n;
    int32_t m;
    int32_t L;
    uint32_t base;
    uint2 key;
    uint32_t* __restrict__ out;           // [n][L][2]
    uint32_t* __restrict__ pool_v;        // scratch [n][m]
    uint64_t* __restrict__ pool_rb;       // scratch [n][m]
    uint32_t* __restrict__ gbias;         // scratch [n][m]: per-slot VertexBias (degree)
    uint64_t* __restrict__ gblk;          // scratch [n_warps][nblk] when shared memory is too small
    int smem_ok;
    int warps_per_block;
    const uint32_t* __restrict__ colc;    // col entries [0, colc_n) on the device (k_mdrw_fast; = col in memory)
    uint64_t colc_n;
    const uint64_t* __restrict__ nmp;     // optional next-vertex metadata per entry (row << 24 | deg)
    unsigned long long* ticket = nullptr; // k_mdrw_fast: instances from a global ticket (zeroed per call)
    const uint4* __restrict__ nrc = nullptr;   // optional next-vertex records {u, deg, row lo, hi} (k_mdrw_fast)
};

__global__ void k_mdrw(MdrwArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = lane_id();
    const int wib = threadIdx.x >> 5;
    const uint32_t m = static_cast<uint32_t>(a.m);
    const uint32_t nblk = (m + 31) / 32;
    // block totals in shared memory (small: all instances fit in one wave); the
    // per-slot biases stay in global memory (one coalesced 128 B read per step)
    uint64_t* blk = a.smem_ok ? reinterpret_cast<uint64_t*>(smem_raw) + static_cast<size_t>(nblk) * wib
                              : a.gblk + global_warp_id() * nblk;
    for (uint64_t w = global_warp_id(); w < a.n; w += total_warps()) {
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        uint32_t* bias = a.gbias + w * m;
        uint32_t* pv = a.pool_v + w * m;
        uint64_t* prb = a.pool_rb + w * m;
        // init pool (slot order = seeds order)
        for (uint32_t s = lane; s < m; s += 32) {
            const uint32_t v = a.seeds[w * m + s];
            const int64_t r0 = __ldg(a.rp + v);
            pv[s] = v;
            prb[s] = static_cast<uint64_t>(r0);
            bias[s] = static_cast<uint32_t>(__ldg(a.rp + v + 1) - r0);
        }
        __syncwarp();
        uint64_t T = 0;
        for (uint32_t b = 0; b < nblk; ++b) {
            const uint32_t s = b * 32 + lane;
            const uint64_t tot = warp_sum(s < m ? bias[s] : 0u);
            if (lane == 0) blk[b] = tot;
            T += tot;
        }
        __syncwarp();
        uint32_t* orow = a.out + w * static_cast<uint64_t>(a.L) * 2;
        uint2 ebuf = make_uint2(NONE, NONE);
        for (int32_t t = 0; t < a.L; ++t) {
            uint32_t v = NONE, u = NONE;
            if (T > 0) {
                const uint64_t x = below(draw_u64(a.key, inst, static_cast<uint32_t>(t), 0u, word3(PURPOSE_VERTEX, 0, 0)), T);
                const uint64_t Ue = draw_u64(a.key, inst, static_cast<uint32_t>(t), 0u, word3(PURPOSE_EDGE, 0, 0));
                // block containing x
                uint64_t base = 0;
                uint32_t bsel = 0;
                uint64_t blo = 0;
                for (uint32_t g0 = 0; g0 < nblk; g0 += 32) {
                    const uint64_t vb = (g0 + lane < nblk) ? blk[g0 + lane] : 0;
                    const uint64_t incl = warp_incl_scan(vb) + base;
                    const unsigned hit = __ballot_sync(FULL, incl > x);
                    if (hit) {
                        const int f = __ffs(hit) - 1;
                        bsel = g0 + f;
                        blo = __shfl_sync(FULL, incl - vb, f);
                        break;
                    }
                    base = __shfl_sync(FULL, incl, 31);
                }
                // the block's biases and pool entries are read together (one round)
                const uint32_t s0 = bsel * 32 + lane;
                const bool in = s0 < m;
                const uint32_t e = in ? bias[s0] : 0u;
                const uint32_t pvl = in ? pv[s0] : NONE;
                const uint64_t prbl = in ? prb[s0] : 0;
                const uint64_t incl2 = warp_incl_scan(static_cast<uint64_t>(e)) + blo;
                const unsigned hit2 = __ballot_sync(FULL, incl2 > x);
                const int fl = __ffs(hit2) - 1;
                const uint32_t slot = bsel * 32 + fl;
                const uint32_t d = __shfl_sync(FULL, e, fl);
                const uint32_t vsel = __shfl_sync(FULL, pvl, fl);
                const uint64_t rb = __shfl_sync(FULL, prbl, fl);
                if (lane == 0) {
                    v = vsel;
                    const uint64_t j = below(Ue, d);
                    u = __ldg(a.col + rb + j);
                    const int64_t ru = __ldg(a.rp + u);
                    const uint32_t du = static_cast<uint32_t>(__ldg(a.rp + u + 1) - ru);
                    pv[slot] = u;
                    prb[slot] = static_cast<uint64_t>(ru);
                    bias[slot] = du;
                    blk[bsel] = blk[bsel] + du - d;
                    T = T + du - d;
                }
                __syncwarp();
                T = __shfl_sync(FULL, T, 0);
                v = __shfl_sync(FULL, v, 0);
                u = __shfl_sync(FULL, u, 0);
            }
            // buffer 16 steps (2 words each) per 32 lanes, flush coalesced
            const int k = t & 15;
            if (lane == 2 * k) ebuf.x = v;
            if (lane == 2 * k + 1) ebuf.x = u;
            if (k == 15 || t == a.L - 1) {
                const int32_t t0 = t & ~15;
                const int32_t idx = t0 * 2 + lane;
                if (idx < (t + 1) * 2) orow[idx] = ebuf.x;
            }
        }
        __syncwarp();
    }
}

// MDRW, pools of m <= 2048 slots (nblk <= 64 blocks of 32): the instruction diet of
// k_mdrw.  Block totals live in registers (lane l: blocks 2l, 2l+1) so the block search
// is one u64 warp scan; a slot's state is one 16 B record {v, bias, row start lo, hi}
// (one load per lane per step); the step's two draws come from a per-lane buffer
// refilled every 32 steps; the neighbour and its row are loaded by every lane (broadcast
// loads) so no lane-0 section and no result shuffles remain.  Same x, same slot, same
// neighbour as k_mdrw and the oracle (bit-identical).
#ifndef MDRW_WARPS_N
#define MDRW_WARPS_N 4
#endif
constexpr int MDRW_WARPS = MDRW_WARPS_N;
#ifndef MDRW_SPEC
#define MDRW_SPEC 0          // guess step t+1's block during step t's metadata load (A/B r02 cfg5: 3.19 vs 2.93 ms off)
#endif
#ifndef MDRW_KEEP_POOL
#define MDRW_KEEP_POOL 0     // pool-state loads / stores with an L2 evict-last policy (A/B r02 cfg5: 2.97 vs 2.91 ms off, same DRAM bytes)
#endif

// L2 evict-last accesses for the per-instance pool state (kept resident against the random
// per-step entry reads, which are evict-first)
__device__ __forceinline__ uint64_t l2_keep_policy() {
    uint64_t pol = 0;
#if MDRW_KEEP_POOL
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
    return pol;
}
__device__ __forceinline__ uint64_t ld_keep(const uint64_t* p, uint64_t pol) {
#if MDRW_KEEP_POOL
    uint64_t v;
    asm volatile("ld.global.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return *p;
#endif
}
__device__ __forceinline__ void st_keep(uint64_t* p, uint64_t v, uint64_t pol) {
#if MDRW_KEEP_POOL
    asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
#else
    (void)pol;
    *p = v;
#endif
}
#ifndef MDRW_PVV_64B
#define MDRW_PVV_64B 1       // the slot's vertex id (output only) with a 64 B L2 fetch
#endif
#ifndef MDRW_STREAM_HINT
#define MDRW_STREAM_HINT 1   // evict-first loads for the per-step random entry + metadata
#endif   // warps per block; 28 warps / SM at 72 registers
__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t v) {
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// kNarrow: a block of 32 slot biases sums below 2^32 (max degree < 2^27): u32 block scan.
// kPacked (max degree < 2^24, E < 2^40): a slot is one u64 {row start << 24 | degree} --
// the same word as the next-vertex metadata -- and the slot's vertex id sits in a separate
// array read only for the output, off the step's dependent chain; the per-step block read
// is 256 B instead of 512 B and the pool state (n x m x 8 B) is more L2-resident.
template <bool kNarrow, bool kPacked>
__global__ void __launch_bounds__(MDRW_WARPS * 32, 28 / MDRW_WARPS) k_mdrw_fast(MdrwArgs a, uint4* __restrict__ pool,
                                                                 uint64_t* __restrict__ prec, uint32_t* __restrict__ pvid) {
    const int lane = lane_id();
    const uint32_t m = static_cast<uint32_t>(a.m);
    for (uint64_t w = walker_ticket(a.ticket); w < a.n; w = walker_ticket(a.ticket)) {
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        uint4* ps = pool + w * m;
        uint64_t* pr = prec + w * m;
        uint32_t* pvv = pvid + w * m;
        // init pool (slot order = seeds order) and the two block totals of this lane
        uint64_t bA = 0, bB = 0;
        for (uint32_t b = 0; b * 32 < m; ++b) {   // block b is held by lane b >> 1
            const uint32_t s = b * 32 + lane;
            uint32_t dv = 0;
            if (s < m) {
                const uint32_t v = a.seeds[w * m + s];
                const int64_t r0 = __ldg(a.rp + v);
                dv = static_cast<uint32_t>(__ldg(a.rp + v + 1) - r0);
                if constexpr (kPacked) {
                    pr[s] = static_cast<uint64_t>(r0) << 24 | dv;
                    pvv[s] = v;
                } else {
                    ps[s] = make_uint4(v, dv, static_cast<uint32_t>(r0), static_cast<uint32_t>(static_cast<uint64_t>(r0) >> 32));
                }
            }
            const uint64_t tot = warp_sum(static_cast<uint64_t>(dv));
            if (lane == static_cast<int>(b >> 1)) { if (b & 1) bB = tot; else bA = tot; }
        }
        // inclusive prefix of the block-pair totals over the lanes, kept up to date by deltas
        // (a step changes one block): the block search is one ballot, no scan
        const uint64_t pol = l2_keep_policy();
        uint64_t pol_ef = 0;
#if MDRW_STREAM_HINT == 2
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_ef));
#endif
        (void)pol_ef;
        uint64_t incl = warp_incl_scan(bA + bB);
        uint64_t T = __shfl_sync(FULL, incl, 31);
        __syncwarp();
        uint32_t* orow = a.out + w * static_cast<uint64_t>(a.L) * 2;
        uint32_t ebuf = NONE;
        uint64_t uxb = 0, ueb = 0;
        // block of x: the pair owner f (ballot over the inclusive pair prefix), then which half
        auto locate = [&](uint64_t x, uint32_t& bsel, uint64_t& blo) {
            const int f = __ffs(__ballot_sync(FULL, incl > x)) - 1;   // exists: x < T
            const uint64_t ex = __shfl_sync(FULL, incl - bA - bB, f);
            const uint64_t fa = __shfl_sync(FULL, bA, f);
            const bool second = x >= ex + fa;
            bsel = 2 * f + (second ? 1 : 0);
            blo = second ? ex + fa : ex;
        };
        // the block's slot records (lane = slot within the block)
        auto load_block = [&](uint32_t bsel, uint64_t& rec, uint4& e) {
            const uint32_t s0 = bsel * 32 + lane;
            if constexpr (kPacked) rec = s0 < m ? ld_keep(pr + s0, pol) : 0;
            else e = s0 < m ? ps[s0] : make_uint4(NONE, 0, 0, 0);
        };
        // step t's block, loaded ahead: at the end of step t-1 the block of step t is
        // requested with the totals before t-1's update (a guess, usually right), so that
        // load overlaps t-1's dependent metadata load; a wrong guess is reloaded
        uint32_t bsel = 0;
        uint64_t blo = 0, rec = 0;
        uint4 e = make_uint4(NONE, 0, 0, 0);
        if (a.L > 0) {
            uxb = draw_u64(a.key, inst, static_cast<uint32_t>(lane), 0u, word3(PURPOSE_VERTEX, 0, 0));
            ueb = draw_u64(a.key, inst, static_cast<uint32_t>(lane), 0u, word3(PURPOSE_EDGE, 0, 0));
            if (T > 0) {
                locate(below(__shfl_sync(FULL, uxb, 0), T), bsel, blo);
                load_block(bsel, rec, e);
            }
        }
        for (int32_t t = 0; t < a.L; ++t) {
            const uint64_t Ue = __shfl_sync(FULL, ueb, t & 31);
            uint32_t v = NONE, u = NONE;
            if (T > 0) {
                const uint64_t x = below(__shfl_sync(FULL, uxb, t & 31), T);
                const uint32_t s0 = bsel * 32 + lane;
                uint32_t bias;
                if constexpr (kPacked) bias = static_cast<uint32_t>(rec & 0xFFFFFFu);
                else bias = e.y;
                uint64_t incl2;
                if constexpr (kNarrow) incl2 = static_cast<uint64_t>(warp_incl_scan_u32(bias)) + blo;
                else incl2 = warp_incl_scan(static_cast<uint64_t>(bias)) + blo;
                const int fl = __ffs(__ballot_sync(FULL, incl2 > x)) - 1;
                const uint32_t d = __shfl_sync(FULL, bias, fl);
                uint64_t rb;
                if constexpr (kPacked) {
                    rb = __shfl_sync(FULL, rec, fl) >> 24;
#if MDRW_PVV_64B
                    v = ld_rand_rw_u32(pvv + bsel * 32 + fl);   // for the output only (not on the next step's chain)
#else
                    v = pvv[bsel * 32 + fl];   // for the output only (not on the next step's chain)
#endif
                } else {
                    v = __shfl_sync(FULL, e.x, fl);
                    rb = static_cast<uint64_t>(__shfl_sync(FULL, e.w, fl)) << 32 | __shfl_sync(FULL, e.z, fl);
                }
                const uint64_t ei = rb + below(Ue, d);
                CSAW_DASSERT(!a.nrc || ei < a.colc_n);
                int64_t ru;
                uint32_t du;
                uint64_t mt = 0;
                // the next step's draws (refilled every 32 steps) and its guessed block
                if (((t + 1) & 31) == 0 && t + 1 < a.L) {
                    uxb = draw_u64(a.key, inst, static_cast<uint32_t>(t + 1 + lane), 0u, word3(PURPOSE_VERTEX, 0, 0));
                    ueb = draw_u64(a.key, inst, static_cast<uint32_t>(t + 1 + lane), 0u, word3(PURPOSE_EDGE, 0, 0));
                }
                uint4 nr = make_uint4(0, 0, 0, 0);
                if (a.nrc) {   // the entry, the new vertex's row and its degree in one 16 B read
                    nr = ld_rand_cs_v4(a.nrc + ei);
                    u = nr.x;
                } else if (a.nmp) {   // the new vertex's row and degree come with the entry (no dependent lookup)
#if MDRW_STREAM_HINT == 2
                    asm volatile("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(mt) : "l"(a.nmp + ei), "l"(pol_ef));
                    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(u) : "l"(a.col + ei), "l"(pol_ef));
#elif MDRW_STREAM_HINT
                    mt = ld_rand_cs_u64(a.nmp + ei);   // read once: evict first, keep the pool state in L2
                    u = ld_rand_cs_u32(a.col + ei);
#else
                    mt = __ldg(a.nmp + ei);
                    u = __ldg(a.col + ei);
#endif
                } else {
                    u = ei < a.colc_n ? __ldg(a.colc + ei) : __ldg(a.col + ei);   // OOM zero-copy: host beyond colc_n
                }
                const uint64_t Uxn = __shfl_sync(FULL, uxb, (t + 1) & 31);
                uint32_t gsel = 0;
                uint64_t glo = 0, grec = 0;
                uint4 ge = make_uint4(NONE, 0, 0, 0);
                if (MDRW_SPEC && t + 1 < a.L) {   // guess with the totals before this step's update
                    locate(below(Uxn, T), gsel, glo);
                    load_block(gsel, grec, ge);
                } else {
                    gsel = NONE;
                }
                if (a.nrc) {
                    ru = static_cast<int64_t>(static_cast<uint64_t>(nr.w) << 32 | nr.z);
                    du = nr.y;
                    mt = static_cast<uint64_t>(ru) << 24 | du;
                } else if (a.nmp) {
                    ru = static_cast<int64_t>(mt >> 24);
                    du = static_cast<uint32_t>(mt & 0xFFFFFFu);
                } else {
                    ru = __ldg(a.rp + u);
                    du = static_cast<uint32_t>(__ldg(a.rp + u + 1) - ru);
                    mt = static_cast<uint64_t>(ru) << 24 | du;
                }
                const uint4 ne = make_uint4(u, du, static_cast<uint32_t>(ru), static_cast<uint32_t>(static_cast<uint64_t>(ru) >> 32));
                if (lane == fl) {
                    if constexpr (kPacked) {
                        st_keep(pr + s0, mt, pol);
                        pvv[s0] = u;
                    } else {
                        ps[s0] = ne;
                    }
                }
                const uint64_t delta = static_cast<uint64_t>(du) - d;   // mod 2^64
                const int owner = static_cast<int>(bsel >> 1);
                if (lane == owner) {
                    if (bsel & 1) bB += delta;
                    else bA += delta;
                }
                if (lane >= owner) incl += delta;
                T += delta;
                __syncwarp();
                if (t + 1 < a.L && T > 0) {   // the real block of step t + 1
                    const uint32_t osel = bsel;
                    locate(below(Uxn, T), bsel, blo);
                    if (bsel == gsel) {
                        rec = grec;
                        e = ge;
                        if (bsel == osel && lane == fl) { rec = mt; e = ne; }   // the guess predates this write
                    } else {
                        load_block(bsel, rec, e);
                    }
                }
            }
            // buffer 16 steps (2 words each) per 32 lanes, flush coalesced
            const int k = t & 15;
            if (lane == 2 * k) ebuf = v;
            if (lane == 2 * k + 1) ebuf = u;
            if (k == 15 || t == a.L - 1) {
                const int32_t t0 = t & ~15;
                const int32_t idx = t0 * 2 + lane;
                if (idx < (t + 1) * 2) orow[idx] = ebuf;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- host launchers
static int walk_grid(const csaw_graph* g, int64_t n) {
    const int64_t warps = std::min<int64_t>(n, static_cast<int64_t>(g->num_sms) * 64);
    return static_cast<int>(std::max<int64_t>(1, (warps + WALK_WARPS - 1) / WALK_WARPS));
}

constexpr int N2X_CHUNKS = 8;   // pipelined host copies of the node2vec index walk (copy_ev holds K + 1 events)
bool walk_path_direct_ok(const csaw_graph* g, const csaw_bias& b) {
    return !(b.kind == CSAW_BIAS_NODE2VEC && g->n2x_rec && !g->w && !g->oom && n2v_integer_scale(b.p, b.q) != 0);
}

csaw_status run_walk(const csaw_graph* g, const csaw_bias& b, int32_t length, const uint32_t* d_seeds, int64_t n,
                     uint64_t base, uint64_t seed, uint32_t* d_path, cudaStream_t st, uint32_t* h_path, bool* copied) {
    if (copied) *copied = false;
    // argument checks before any statistics / timing state is recorded
    if (b.kind == CSAW_BIAS_NODE2VEC && !g->rows_sorted)
        return fail(CSAW_ERR_BAD_GRAPH, "node2vec needs sorted CSR rows (N(prev) membership)");
    if (b.kind == CSAW_BIAS_WEIGHT && !g->w)
        return fail(CSAW_ERR_INVALID_ARG, "CSAW_BIAS_WEIGHT needs a graph created with edge weights");
    void* cnt;
    CSAW_TRY(g->scratch.get(SL_COUNTS, 64, &cnt));
    CSAW_CUDA(cudaMemsetAsync(cnt, 0, 64, st));
    CSAW_TRY(stats_begin(g, st));
    CSAW_TRY(hot_begin(g, st));
    note_launch();
    const uint2 key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    // zero-copy OOM mode: col_idx is read in place from pinned host memory (UVA)
    const uint32_t* colp = g->col ? g->col : g->oomst.src_col;
    WalkArgs a{g->row_ptr, colp, g->deg, d_seeds, static_cast<uint64_t>(n), length,
               static_cast<uint32_t>(base), key, d_path, static_cast<unsigned long long*>(cnt), g->ccache};
    if (b.kind == CSAW_BIAS_WEIGHT && g->gbw) {
        constexpr int hw = 2;
        const int64_t hwarps = std::min<int64_t>(n, static_cast<int64_t>(g->num_sms) * 64);
        k_walk_gbw<<<static_cast<int>((hwarps + hw - 1) / hw), hw * 32, 0, st>>>(a, g->gbw, g->gwmeta, g->cpsw, g->w,
                                                                                   g->gbw_buckets);
    } else if (b.kind == CSAW_BIAS_DEGREE && g->gbk) {
        constexpr int hw = GB_WARPS;   // warps per block: the few walkers (cfg2: 4,000 warps) spread over all SMs
        const int64_t hwarps = std::min<int64_t>(n, static_cast<int64_t>(g->num_sms) * 64);
        k_walk_gb<<<static_cast<int>((hwarps + hw - 1) / hw), hw * 32, 0, st>>>(a, g->gbk, g->gmeta, g->cps,
                                                                                     static_cast<uint64_t>(g->E), g->gb_buckets);
    } else if (b.kind == CSAW_BIAS_DEGREE && g->wix_leaf) {
        // group kernels: 2-warp blocks, so few walkers (cfg2: 1,000 warps) still spread over all SMs
        const int wpb = g->wix_group == 32 ? WALK_WARPS : 2;
        const int blk = wpb * 32;
        const int64_t walkers_per_warp = 32 / g->wix_group;
        const int64_t warps = std::min<int64_t>((n + walkers_per_warp - 1) / walkers_per_warp,
                                                static_cast<int64_t>(g->num_sms) * 64);
        const int grid = static_cast<int>(std::max<int64_t>(1, (warps + wpb - 1) / wpb));
        const uint4* rec = g->wrec;
        if (g->wix_group == 32 && g->whead) {
            // small blocks spread the few walkers evenly over the SMs (cfg2: 4,000 warps on 148 SMs)
            constexpr int hw = 2;   // warps per block (A/B cfg2: 1: 2.46, 2: 2.43, 4: 2.44, 8: 2.48 ms)
            const int64_t hwarps = std::min<int64_t>(n, static_cast<int64_t>(g->num_sms) * 64);
            const int hg = static_cast<int>((hwarps + hw - 1) / hw);
            if (g->wix_leaf == 32) k_walk_head<32><<<hg, hw * 32, 0, st>>>(a, g->whead, g->c32, g->wcol, g->winn);
            else if (g->wix_leaf == 128) k_walk_head<128><<<hg, hw * 32, 0, st>>>(a, g->whead, g->c32, g->wcol, g->winn);
            else k_walk_head<64><<<hg, hw * 32, 0, st>>>(a, g->whead, g->c32, g->wcol, g->winn);
        } else if (g->wix_group == 32) {
            if (g->wix_leaf == 32) k_walk_wix<32><<<grid, blk, 0, st>>>(a, rec, g->c32, g->wcol, g->winn);
            else if (g->wix_leaf == 64) k_walk_wix<64><<<grid, blk, 0, st>>>(a, rec, g->c32, g->wcol, g->winn);
            else k_walk_wix<128><<<grid, blk, 0, st>>>(a, rec, g->c32, g->wcol, g->winn);
        } else if (g->wix_group == 16) {
            if (g->wix_leaf == 64) k_walk_wixg<16, 64><<<grid, blk, 0, st>>>(a, rec, g->c32, g->wcol, g->winn);
            else k_walk_wixg<16, 128><<<grid, blk, 0, st>>>(a, rec, g->c32, g->wcol, g->winn);
        } else {
            if (g->wix_leaf == 32) k_walk_wixg<8, 32><<<grid, blk, 0, st>>>(a, rec, g->c32, g->wcol, g->winn);
            else if (g->wix_leaf == 64) k_walk_wixg<8, 64><<<grid, blk, 0, st>>>(a, rec, g->c32, g->wcol, g->winn);
            else k_walk_wixg<8, 128><<<grid, blk, 0, st>>>(a, rec, g->c32, g->wcol, g->winn);
        }
    } else if (b.kind == CSAW_BIAS_DEGREE && g->cps) {
        k_walk_cached<<<walk_grid(g, n), WALK_WARPS * 32, 0, st>>>(a, g->cps, g->bt, g->bt_off, g->nmp);
    } else if ((b.kind == CSAW_BIAS_DEGREE && g->ebias) || b.kind == CSAW_BIAS_WEIGHT) {
        // per-edge bias streams (vscan.cuh): the materialised degree bias or the edge weights
        CSAW_TRY(launch_walk_vscan(g, b.kind == CSAW_BIAS_WEIGHT, d_seeds, static_cast<uint64_t>(n), length,
                                   static_cast<uint32_t>(base), key, d_path, static_cast<unsigned long long*>(cnt), 0,
                                   st));
    } else if (b.kind == CSAW_BIAS_DEGREE) {
        k_walk<false><<<walk_grid(g, n), WALK_WARPS * 32, 0, st>>>(a);
    } else if (b.kind == CSAW_BIAS_UNIFORM) {
        k_walk<true><<<walk_grid(g, n), WALK_WARPS * 32, 0, st>>>(a);
    } else if (b.kind == CSAW_BIAS_MH) {
        k_walk_variant<CSAW_BIAS_MH><<<walk_grid(g, n), WALK_WARPS * 32, 0, st>>>(a, 0, g->V);
    } else if (b.kind == CSAW_BIAS_RESTART || b.kind == CSAW_BIAS_JUMP) {
        const uint64_t theta = static_cast<uint64_t>(std::floor(b.pf * 4294967296.0));
        if (b.kind == CSAW_BIAS_RESTART) k_walk_variant<CSAW_BIAS_RESTART><<<walk_grid(g, n), WALK_WARPS * 32, 0, st>>>(a, theta, g->V);
        else k_walk_variant<CSAW_BIAS_JUMP><<<walk_grid(g, n), WALK_WARPS * 32, 0, st>>>(a, theta, g->V);
    } else if (b.kind == CSAW_BIAS_NODE2VEC) {
        N2vArgs na;
        na.wa = a;
        const uint32_t m = n2v_integer_scale(b.p, b.q);
        na.wint[0] = m ? static_cast<uint32_t>(static_cast<double>(m) / b.p) : 0;
        na.wint[1] = m;
        na.wint[2] = m ? static_cast<uint32_t>(static_cast<double>(m) / b.q) : 0;
        na.wf[0] = static_cast<float>(1.0 / b.p);
        na.wf[1] = 1.0f;
        na.wf[2] = static_cast<float>(1.0 / b.q);
        na.ew = g->w;   // weighted graph: b = alpha * w(e) (R33), always the float path
        if (g->w) k_node2vec<true><<<walk_grid(g, n), WALK_WARPS * 32, 0, st>>>(na);
        else if (m && g->n2x_rec && na.wint[0] < (1u << 30) && na.wint[1] < (1u << 30) && na.wint[2] < (1u << 30)) {
            // a pinned host path: N2X_CHUNKS launches over consecutive walker ranges, each range's
            // rows copied back on g->copy_st while the next range walks (the host link, not the
            // walk, bounds an end-to-end call: cfg3 moves 618 MB of paths)
            const bool pipe = h_path && n >= 8 * N2X_CHUNKS * 32;
            if (pipe && !g->copy_st) {
                CSAW_CUDA(cudaStreamCreateWithFlags(&g->copy_st, cudaStreamNonBlocking));
                for (cudaEvent_t& e : g->copy_ev) CSAW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            }
            const int K = pipe ? N2X_CHUNKS : 1;
            const uint64_t row = static_cast<uint64_t>(length) + 1;
            for (int c = 0; c < K; ++c) {
                const uint64_t lo = static_cast<uint64_t>(n) * c / K, hi = static_cast<uint64_t>(n) * (c + 1) / K;
                if (c > 0) CSAW_CUDA(cudaMemsetAsync(static_cast<unsigned long long*>(cnt) + 7, 0, 8, st));   // group ticket
                CSAW_TRY(launch_node2vec_index(g, d_seeds + lo, hi - lo, length, static_cast<uint32_t>(base + lo), key,
                                               d_path + lo * row, static_cast<unsigned long long*>(cnt), na.wint[0],
                                               na.wint[1], na.wint[2], st));
                if (pipe) {
                    CSAW_CUDA(cudaEventRecord(g->copy_ev[c], st));
                    CSAW_CUDA(cudaStreamWaitEvent(g->copy_st, g->copy_ev[c], 0));
                    CSAW_CUDA(cudaMemcpyAsync(h_path + lo * row, d_path + lo * row, sizeof(uint32_t) * (hi - lo) * row,
                                              cudaMemcpyDeviceToHost, g->copy_st));
                }
            }
            if (pipe) {
                CSAW_CUDA(cudaEventRecord(g->copy_ev[N2X_CHUNKS], g->copy_st));
                CSAW_CUDA(cudaStreamWaitEvent(st, g->copy_ev[N2X_CHUNKS], 0));
                if (copied) *copied = true;
            }
        }
        else if (m && g->tri) k_node2vec_tri<<<walk_grid(g, n), N2T_WARPS * 32, 0, st>>>(na, g->tri);
        else if (m) k_node2vec<false><<<walk_grid(g, n), WALK_WARPS * 32, 0, st>>>(na);
        else k_node2vec<true><<<walk_grid(g, n), WALK_WARPS * 32, 0, st>>>(na);
    } else if (b.kind == CSAW_BIAS_MDRW) {
        const uint32_t m = static_cast<uint32_t>(b.pool_size);
        const uint32_t nblk = (m + 31) / 32;
        if (nblk <= 64 && !(g->flags & CSAW_GRAPH_MDRW_GENERIC)) {   // pools up to 2,048 slots (cfg5: 2,000)
            // slot records: 16 B {v, degree, row} (the slot's vertex comes with the block, no separate
            // vertex-id read per step: cfg5 with next-vertex records 2.61 vs 2.76 ms packed); with
            // CSAW_GRAPH_MDRW_ALT_RECORDS 8 B packed {row << 24 | degree} + a u32 vertex-id array (A/B)
            const bool alt = (g->flags & CSAW_GRAPH_MDRW_ALT_RECORDS) != 0;
            const bool packed = g->max_deg < (int64_t(1) << 24) && g->E < (int64_t(1) << 40) && alt;
            void *pool = nullptr, *pvid = nullptr;
            if (packed) {
                CSAW_TRY(g->scratch.get(SL_TMP0, sizeof(uint64_t) * n * m, &pool));
                CSAW_TRY(g->scratch.get(SL_TMP1, sizeof(uint32_t) * n * m, &pvid));
            } else {
                CSAW_TRY(g->scratch.get(SL_TMP0, sizeof(uint4) * n * m, &pool));
            }
            MdrwArgs ma{g->row_ptr, colp, d_seeds, static_cast<uint64_t>(n), b.pool_size, length,
                        static_cast<uint32_t>(base), key, d_path, nullptr, nullptr, nullptr, nullptr, 0, WALK_WARPS,
                        g->col ? g->col : g->oomst.d_colc,
                        static_cast<uint64_t>(g->col ? g->E : g->oomst.colc_n), g->col ? g->nmp : nullptr};
            const int64_t warps = std::min<int64_t>(n, static_cast<int64_t>(g->num_sms) * 28);
            const int mg = static_cast<int>((warps + MDRW_WARPS - 1) / MDRW_WARPS);
            uint4* p4 = static_cast<uint4*>(pool);
            uint64_t* p8 = static_cast<uint64_t*>(pool);
            uint32_t* pv = static_cast<uint32_t*>(pvid);
            const bool narrow = g->max_deg < (int64_t(1) << 27);
            ma.ticket = static_cast<unsigned long long*>(cnt) + 7;   // zeroed with the counters
            ma.nrc = g->col ? g->nrec : nullptr;
            if (packed && narrow) k_mdrw_fast<true, true><<<mg, MDRW_WARPS * 32, 0, st>>>(ma, p4, p8, pv);
            else if (packed) k_mdrw_fast<false, true><<<mg, MDRW_WARPS * 32, 0, st>>>(ma, p4, p8, pv);
            else if (narrow) k_mdrw_fast<true, false><<<mg, MDRW_WARPS * 32, 0, st>>>(ma, p4, p8, pv);
            else k_mdrw_fast<false, false><<<mg, MDRW_WARPS * 32, 0, st>>>(ma, p4, p8, pv);
            CSAW_CUDA(cudaGetLastError());
            CSAW_TRY(hot_end(g, st));
            CSAW_TRY(stats_end(g, st));
            g->stats.sampled_edges = static_cast<uint64_t>(n) * length;
            g->pending_counters = static_cast<const unsigned long long*>(cnt);
            return CSAW_OK;
        }
        const size_t per = static_cast<size_t>(nblk) * 8;
        int wpb = static_cast<int>(std::min<size_t>(8, (200 * 1024) / std::max<size_t>(per, 1)));
        const bool smem_ok = wpb >= 1;
        if (!smem_ok) wpb = 8;
        const int64_t max_warps = static_cast<int64_t>(g->num_sms) * 64;
        const int64_t warps = std::min<int64_t>(n, max_warps);
        const int grid = static_cast<int>((warps + wpb - 1) / wpb);
        void *pv, *prb, *gb = nullptr, *gk = nullptr;
        CSAW_TRY(g->scratch.get(SL_TMP0, sizeof(uint32_t) * n * m, &pv));
        CSAW_TRY(g->scratch.get(SL_TMP1, sizeof(uint64_t) * n * m, &prb));
        CSAW_TRY(g->scratch.get(SL_TMP2, sizeof(uint32_t) * n * m, &gb));
        const size_t smem = smem_ok ? per * wpb : 0;
        if (!smem_ok) {
            CSAW_TRY(g->scratch.get(SL_GLIST, sizeof(uint64_t) * nblk * grid * wpb, &gk));
        } else {
            CSAW_CUDA(cudaFuncSetAttribute(k_mdrw, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        }
        MdrwArgs ma{g->row_ptr, colp, d_seeds, static_cast<uint64_t>(n), b.pool_size, length,
                    static_cast<uint32_t>(base), key, d_path, static_cast<uint32_t*>(pv),
                    static_cast<uint64_t*>(prb), static_cast<uint32_t*>(gb), static_cast<uint64_t*>(gk),
                    smem_ok ? 1 : 0, wpb, nullptr, 0, nullptr};
        k_mdrw<<<grid, wpb * 32, smem, st>>>(ma);
    } else {
        return fail(CSAW_ERR_INVALID_ARG, "bias kind is not a walk selector");
    }
    CSAW_CUDA(cudaGetLastError());
    CSAW_TRY(hot_end(g, st));
    CSAW_TRY(stats_end(g, st));
    g->stats.sampled_edges = static_cast<uint64_t>(n) * length;   // L edges per walker / instance (R30)
    g->pending_counters = static_cast<const unsigned long long*>(cnt);
    return CSAW_OK;
}

}  // namespace csaw
