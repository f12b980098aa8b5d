// vscan.cuh — per-edge bias streams: vectorised CTPS scans for EdgeBias = f(e)
// (Eq. 3) read from an array aligned with col_idx.
//
// Two element types share one engine:
//   float    -- caller edge weights (csaw_csr.weights): the float path of reading R28,
//               fp32 biases accumulated in fp64, draw x = r * T with r = (U >> 11) 2^-53;
//   uint32_t -- a materialised integer bias per CSR entry (deg(col[e]) for the degree
//               bias, CSAW_GRAPH_EDGE_BIAS): exact u64 CTPS, x = below(U, T), bit-identical
//               to the gather scan of select.cuh and to the oracle.
// The pool is read as 16 B vectors (4 entries per lane, 128 per warp row, VU rows in
// flight), aligned down to the vector containing the pool's first entry; entries
// outside the pool read as 0.  The arrays carry >= 128 entries of zero padding.
//
// CTPS layout (shared memory, Acc[TAB] per pool): rows are grouped in chunks of
// m = max(VMIN, ceil(nrows / TAB)) rows (rounded up to whole batches of VU); tab[c] = the cumulative total at the end of chunk
// c (lane accumulators over the chunk's rows, one warp reduction per chunk, then a prefix
// over the chunks).  The chunking depends only on the pool (its first entry and length),
// never on how many warps build it, so every launch shape gives the same sums (R7).  A
// search finds the chunk holding x in the table and rescans it row by row (lane prefix of
// 4 entries + Kogge-Stone across lanes): two-level ITS.
//
// Float rounding (R28): those association orders differ from the oracle's left-to-right
// fp64 sum by a few ulps -- picks may differ only for draws within that distance of a
// boundary, far inside the checker's 1e-6 rule (a rescan that finds no boundary above x in
// its chunk, possible only through rounding, continues into the next).  Zero-weight regions are never chosen (R4): the search
// takes the first entry with b > 0 and S_{i+1} > x; a draw at or beyond every boundary
// (possible only through rounding) takes the last positive entry.
#pragma once

#include "common.cuh"
#include "select.cuh"

namespace csaw {

constexpr int VROW = 128;   // pool entries per row (one 16 B vector per lane)
#ifndef VSCAN_VU
#define VSCAN_VU 4   // A/B r02 cfg2: VU 8 59.4 ms (register spills) vs 4: 44.4 ms
#endif
#ifndef VSCAN_PREFETCH
#define VSCAN_PREFETCH 0   // A/B r02 cfg2: bulk L2 prefetch of the pool 48.4 ms, without 47.3 ms (hub pools sit in L2)
#endif
constexpr int VU = VSCAN_VU;   // rows in flight per warp (VU x 512 B)
#ifndef VSCAN_VMIN
#define VSCAN_VMIN 8   // A/B r02 cfg2: 1 row 114, 4 rows 48.4, 8 rows 44.4 ms
#endif
constexpr int VMIN = VSCAN_VMIN;   // rows per chunk at least (a search rescans one chunk)

template <class E>
struct VTraits;
template <>
struct VTraits<float> {
    using Acc = double;
    using Vec = float4;
    __device__ static __forceinline__ double draw(uint64_t U, double M) {
        const double r = static_cast<double>(U >> 11) * (1.0 / 9007199254740992.0);
        return r * M;
    }
    __device__ static __forceinline__ double val(float e) { return static_cast<double>(e); }
    __device__ static __forceinline__ double sum(double v) {   // butterfly warp reduction (fixed order)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        return v;
    }
    __device__ static __forceinline__ double scan(double v) {   // inclusive Kogge-Stone
        const int lane = lane_id();
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(FULL, v, o);
            if (lane >= o) v += y;
        }
        return v;
    }
};
template <>
struct VTraits<uint32_t> {
    using Acc = uint64_t;
    using Vec = uint4;
    __device__ static __forceinline__ uint64_t draw(uint64_t U, uint64_t M) { return below(U, M); }
    __device__ static __forceinline__ uint64_t val(uint32_t e) { return e; }
    __device__ static __forceinline__ uint64_t sum(uint64_t v) { return warp_sum(v); }
    __device__ static __forceinline__ uint64_t scan(uint64_t v) { return warp_incl_scan(v); }
};

template <class E>
struct VPool {
    using Tr = VTraits<E>;
    using Acc = typename Tr::Acc;
    const E* __restrict__ b;             // per-edge biases (aligned with col)
    const uint32_t* __restrict__ col;
    uint64_t beg;                        // CSR index of the pool's first entry
    uint32_t n;                          // pool size
    uint32_t head;                       // beg mod 4: entries of the first vector before the pool
    uint32_t nrows;

    __device__ __forceinline__ void init(const E* bb, const uint32_t* c, uint64_t b0, uint32_t nn) {
        b = bb; col = c; beg = b0; n = nn;
        head = static_cast<uint32_t>(b0 & 3u);
        nrows = (head + nn + VROW - 1) / VROW;
    }
    // the lane's 4 entries of row r (pool indices r*128 + 4 lane + j - head); 0 outside the pool
    __device__ __forceinline__ void load(uint32_t r, E (&e)[4]) const {
        const auto* vp = reinterpret_cast<const typename Tr::Vec*>(b + (beg - head)) + static_cast<uint64_t>(r) * 32 + lane_id();
        if (r * VROW >= head && (r + 1) * VROW <= head + n) {   // interior row (warp-uniform): no masks
            const typename Tr::Vec q = __ldg(vp);
            e[0] = q.x; e[1] = q.y; e[2] = q.z; e[3] = q.w;
            return;
        }
        const int64_t i0 = static_cast<int64_t>(r) * VROW + 4 * lane_id() - head;
        typename Tr::Vec q;
        if (i0 + 3 >= 0 && i0 < static_cast<int64_t>(n)) q = __ldg(vp);
        else q = typename Tr::Vec{};
        e[0] = q.x; e[1] = q.y; e[2] = q.z; e[3] = q.w;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (i0 + j < 0 || i0 + j >= static_cast<int64_t>(n)) e[j] = E(0);
    }
    __device__ __forceinline__ uint32_t item(uint32_t s) const { return __ldg(col + beg + s); }
    __device__ __forceinline__ E bias(uint32_t s) const { return __ldg(b + beg + s); }
    // Rows [r0, r1) requested into L2 at once by one bulk (TMA) prefetch per 64 KB
    // (cp.async.bulk.prefetch.L2): the whole stretch is in flight while the warp's
    // vector loads walk through it, instead of VU rows at a time.
    __device__ __forceinline__ void prefetch_l2(uint32_t r0, uint32_t r1) const {
#if VSCAN_PREFETCH
        if (lane_id() == 0 && r1 > r0) {
            const char* p = reinterpret_cast<const char*>(b + (beg - head)) + static_cast<uint64_t>(r0) * VROW * sizeof(E);
            uint64_t bytes = static_cast<uint64_t>(r1 - r0) * VROW * sizeof(E);
            while (bytes > 0) {
                const uint32_t sz = static_cast<uint32_t>(bytes < 65536 ? bytes : 65536);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(sz) : "memory");
                p += sz;
                bytes -= sz;
            }
        }
#else
        (void)r0; (void)r1;
#endif
    }
};

template <class E>
struct VCtps {
    typename VTraits<E>::Acc T;
    uint32_t m;          // rows per chunk
    uint32_t nch;        // chunks (table entries)
    uint32_t npos;       // entries with b > 0
    uint32_t lastpos;    // last entry with b > 0 (NONE if npos == 0)
};

template <class E>
struct VRegion {
    uint32_t s;
    typename VTraits<E>::Acc lo;   // S_s
    typename VTraits<E>::Acc b;    // b_s
    uint32_t item;
};

// Scratch shared by the G warps that build one pool together.
template <class E>
struct VGroupShared {
    typename VTraits<E>::Acc T;
    uint32_t npos[8];
    uint32_t last[8];
    uint32_t word;       // broadcast slot (the step's pick)
};

// One row: lane partial sums c[j] = b_0 + .. + b_j (left to right), the row's lane-inclusive
// scan and its total (Kogge-Stone total = lane 31 of the scan).
template <class E>
struct VRow {
    typename VTraits<E>::Acc c[4];
    typename VTraits<E>::Acc incl;
    typename VTraits<E>::Acc tot;
    __device__ __forceinline__ void compute(const E (&e)[4]) {
        using Tr = VTraits<E>;
        c[0] = Tr::val(e[0]);
        c[1] = c[0] + Tr::val(e[1]);
        c[2] = c[1] + Tr::val(e[2]);
        c[3] = c[2] + Tr::val(e[3]);
        incl = Tr::scan(c[3]);
        tot = __shfl_sync(FULL, incl, 31);
    }
};

// Build the chunk table (warp gw of a G-warp group; bar() synchronises the group).
// kCount: also count the positive entries (npos, lastpos) -- needed without replacement;
// a walk needs only T (npos = T > 0, lastpos found on demand).
template <class E, int G, bool kCount = true, class Bar>
__device__ __forceinline__ VCtps<E> vscan_build(const VPool<E>& P, typename VTraits<E>::Acc* __restrict__ tab,
                                                VGroupShared<E>* sh, int gw, Bar&& bar) {
    using Acc = typename VTraits<E>::Acc;
    const int lane = lane_id();
    VCtps<E> C;
    C.m = max(static_cast<uint32_t>(VMIN), (P.nrows + TAB - 1) / TAB);
    C.m = (C.m + VU - 1) / VU * VU;   // whole batches per chunk
    C.nch = (P.nrows + C.m - 1) / C.m;
    uint32_t npos = 0, last1 = 0;   // last1 = last positive index + 1 (0: none)
    __syncwarp();   // the previous pool's readers of tab are done before it is rewritten
    // phase 1: chunk totals; warp gw takes the contiguous chunks [c0, c1), rows in batches
    // of VU (m is a multiple of VU).  Each lane accumulates its entries (left to right within its
    // 4, then row after row); one warp reduction per chunk -- a row costs a vector load and
    // four adds, no shuffles
    const uint32_t c0 = (C.nch * gw) / G, c1 = (C.nch * (gw + 1)) / G;
    const uint32_t rb = c0 * C.m, re = min(P.nrows, c1 * C.m);
    if (re - rb > VU) P.prefetch_l2(rb + VU, re);   // the first VU rows are loaded right away
    uint32_t pl = 0, ll = 0;
    for (uint32_t c = c0; c < c1; ++c) {
        const uint32_t r1 = min(P.nrows, (c + 1) * C.m);
        Acc lacc = 0;
        for (uint32_t r0 = c * C.m; r0 < r1; r0 += VU) {
            E e[VU][4];
#pragma unroll
            for (int u = 0; u < VU; ++u)
                if (r0 + u < r1) P.load(r0 + u, e[u]);
#pragma unroll
            for (int u = 0; u < VU; ++u) {
                if (r0 + u < r1) {
                    using Tr = VTraits<E>;
                    lacc += ((Tr::val(e[u][0]) + Tr::val(e[u][1])) + Tr::val(e[u][2])) + Tr::val(e[u][3]);
                    if constexpr (kCount) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if (e[u][j] > E(0)) {
                                ++pl;
                                ll = (r0 + u) * VROW + 4 * lane + j - P.head + 1;
                            }
                        }
                    }
                }
            }
        }
        const Acc tot = VTraits<E>::sum(lacc);
        if (lane == 0) tab[c] = tot;
    }
    if constexpr (kCount) {
        npos = __reduce_add_sync(FULL, pl);
        last1 = __reduce_max_sync(FULL, ll);
    }
    if constexpr (G > 1) {
        if (lane == 0) { sh->npos[gw] = npos; sh->last[gw] = last1; }
        bar();
    } else {
        __syncwarp();
    }
    // phase 2 (warp 0): cumulative table; lane l owns entries [8 l, 8 l + 8)
    if (gw == 0) {
        Acc loc[8];
        Acc run = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t c = 8 * lane + k;
            if (c < C.nch) run += tab[c];
            loc[k] = run;
        }
        const Acc inc = VTraits<E>::scan(run);
        Acc exf = __shfl_up_sync(FULL, inc, 1);   // exclusive: the previous lane's inclusive total
        if (lane == 0) exf = 0;
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t c = 8 * lane + k;
            if (c < C.nch) tab[c] = exf + loc[k];
        }
        if constexpr (G > 1) {
            if (lane == 0) {
                uint32_t np = 0, l1 = 0;
                for (int k = 0; k < G; ++k) { np += sh->npos[k]; l1 = max(l1, sh->last[k]); }
                sh->npos[0] = np;
                sh->last[0] = l1;
            }
        }
    }
    if constexpr (G > 1) {
        bar();
        npos = sh->npos[0];
        last1 = sh->last[0];
    } else {
        __syncwarp();
    }
    C.T = tab[C.nch - 1];
    if constexpr (kCount) {
        C.npos = npos;
        C.lastpos = last1 ? last1 - 1 : NONE;
    } else {
        C.npos = C.T > 0 ? 1u : 0u;   // "some positive entry" (biases are >= 0)
        C.lastpos = NONE;              // vscan_find locates it if ever needed
    }
    return C;
}

// Region of pool entry s (rescan of its chunk up to its row); warp-collective.
template <class E>
__device__ __forceinline__ VRegion<E> vscan_region_at(const VPool<E>& P, const VCtps<E>& C,
                                                      const typename VTraits<E>::Acc* __restrict__ tab, uint32_t s) {
    using Acc = typename VTraits<E>::Acc;
    const uint32_t rs = (s + P.head) / VROW;
    const uint32_t c = rs / C.m;
    Acc base = c ? tab[c - 1] : 0;
    for (uint32_t r = c * C.m; r < rs; ++r) {
        E e[4];
        P.load(r, e);
        VRow<E> row;
        row.compute(e);
        base += row.tot;
    }
    E e[4];
    P.load(rs, e);
    VRow<E> row;
    row.compute(e);
    Acc ex = __shfl_up_sync(FULL, row.incl, 1);
    if (lane_id() == 0) ex = 0;
    const uint32_t q = (s + P.head) % VROW;
    const int fl = static_cast<int>(q / 4), j = static_cast<int>(q % 4);
    const Acc p0 = base + ex;
    const Acc lo_l = j == 0 ? p0 : p0 + (j == 1 ? row.c[0] : j == 2 ? row.c[1] : row.c[2]);
    VRegion<E> R;
    R.s = s;
    R.lo = __shfl_sync(FULL, lo_l, fl);
    R.b = VTraits<E>::val(P.bias(s));
    R.item = P.item(s);
    return R;
}

// Inverse transform search for a warp-uniform x: the first entry with b > 0 and
// S_{i+1} > x (R4); past every boundary: the last positive entry.  Warp-collective.
template <class E>
__device__ __forceinline__ VRegion<E> vscan_find(const VPool<E>& P, const VCtps<E>& C,
                                                 const typename VTraits<E>::Acc* __restrict__ tab,
                                                 typename VTraits<E>::Acc x) {
    using Acc = typename VTraits<E>::Acc;
    const int lane = lane_id();
    uint32_t lo = 0, hi = C.nch;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (tab[mid] > x) hi = mid; else lo = mid + 1;
    }
    if (lo < C.nch) {
        Acc base = lo ? tab[lo - 1] : 0;
        uint32_t rend = min(P.nrows, (lo + 1) * C.m);   // the chunk; past it only through rounding
        for (uint32_t r0 = lo * C.m; r0 < rend;) {
            const uint32_t nb = min(static_cast<uint32_t>(VU), rend - r0);
            E e[VU][4];
#pragma unroll
            for (int u = 0; u < VU; ++u)
                if (static_cast<uint32_t>(u) < nb) P.load(r0 + u, e[u]);
#pragma unroll
            for (int u = 0; u < VU; ++u) {
                if (static_cast<uint32_t>(u) < nb) {
                    VRow<E> row;
                    row.compute(e[u]);
                    Acc ex = __shfl_up_sync(FULL, row.incl, 1);
                    if (lane == 0) ex = 0;
                    const Acc p0 = base + ex;
                    int jh = -1;
                    Acc lo_h = 0;
#pragma unroll
                    for (int j = 3; j >= 0; --j) {
                        if (e[u][j] > E(0) && p0 + row.c[j] > x) { jh = j; lo_h = j ? p0 + row.c[j - 1] : p0; }
                    }
                    const unsigned hit = __ballot_sync(FULL, jh >= 0);
                    if (hit) {
                        const int f = __ffs(hit) - 1;
                        const int j = __shfl_sync(FULL, jh, f);
                        VRegion<E> R;
                        R.s = (r0 + u) * VROW + 4 * f + j - P.head;
                        R.lo = __shfl_sync(FULL, lo_h, f);
                        R.b = VTraits<E>::val(__shfl_sync(FULL, e[u][j], f));
                        R.item = P.item(R.s);
                        return R;
                    }
                    base += row.tot;
                }
            }
            r0 += nb;
            if (r0 == rend) rend = P.nrows;
        }
    }
    uint32_t last = C.lastpos;
    if (last == NONE) {   // walks: the last positive entry, by a backwards row scan (rounding only)
        for (int32_t r = static_cast<int32_t>(P.nrows) - 1; r >= 0 && last == NONE; --r) {
            E e[4];
            P.load(static_cast<uint32_t>(r), e);
            int jl = -1;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (e[j] > E(0)) jl = j;
            const unsigned hp = __ballot_sync(FULL, jl >= 0);
            if (hp) {
                const int f = 31 - __clz(hp);
                last = static_cast<uint32_t>(r) * VROW + 4 * f + __shfl_sync(FULL, jl, f) - P.head;
            }
        }
    }
    return vscan_region_at(P, C, tab, last);
}

// With replacement (walks): one draw, x = draw(U, T).
template <class E>
__device__ __forceinline__ uint32_t vscan_select_wr(const VPool<E>& P, const VCtps<E>& C,
                                                    const typename VTraits<E>::Acc* __restrict__ tab, uint64_t U) {
    if (C.npos == 0) return NONE;
    return vscan_find(P, C, tab, VTraits<E>::draw(U, C.T)).item;
}

// Without replacement (sampling): k distinct picks with bipartite region search (box steps
// 1-5; R1 fresh draw; R2 cap a_max then exact updated sampling), the same draw
// sequence as select.cuh's select_wor and oracle_select_wor(_float).  Picks are resolved one
// after another (pick j sees picks < j, R3) with the warp sharing every search: pick q < 32
// is held by lane q, later picks in glist (>= k entries, required when k > 32).  emit(rank,
// s, item) is called once per pick in ascending pool order (R11).
template <class E, class Emit>
__device__ uint32_t vscan_select_wor(const VPool<E>& P, const VCtps<E>& C, const typename VTraits<E>::Acc* tab,
                                     uint32_t k, DrawKey& dk, uint32_t a_max, PickRec* __restrict__ glist,
                                     Emit&& emit) {
    using Tr = VTraits<E>;
    using Acc = typename Tr::Acc;
    const int lane = lane_id();
    if (k == 0 || C.npos == 0) return 0;
    if (k >= C.npos) {   // select all positive entries, ascending (R8)
        uint32_t rank = 0;
        for (uint32_t r = 0; r < P.nrows; ++r) {
            E e[4];
            P.load(r, e);
            uint32_t pl = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) pl += e[j] > E(0);
            uint32_t ex = pl;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, ex, o);
                if (lane >= o) ex += y;
            }
            const uint32_t tot = __shfl_sync(FULL, ex, 31);
            uint32_t rk = rank + ex - pl;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (e[j] > E(0)) {
                    const uint32_t s = r * VROW + 4 * lane + j - P.head;
                    emit(rk++, s, P.item(s));
                }
            }
            rank += tot;
        }
        return C.npos;
    }
    const Acc T = C.T;
    uint32_t mine = NONE;   // lane q: pick q
    auto taken = [&](uint32_t s, uint32_t j) -> bool {   // s warp-uniform; picks [0, j) made
        if (__ballot_sync(FULL, static_cast<uint32_t>(lane) < min(j, 32u) && mine == s)) return true;
        for (uint32_t q = 32; q < j; ++q)
            if (glist[q].s == s) return true;
        return false;
    };
    // exact updated sampling (Fig. 6(b)): the CTPS over the untaken entries (taken ones
    // masked to 0), searched at draw(U, T'); pool order, same row structure
    auto updated = [&](uint32_t j, uint64_t U) -> uint32_t {
        auto masked = [&](uint32_t r, E (&e)[4]) {
            P.load(r, e);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const uint32_t s = r * VROW + 4 * lane + jj - P.head;
                bool t = false;
                for (uint32_t q = 0; q < min(j, 32u); ++q) t |= __shfl_sync(FULL, mine, q) == s;
                for (uint32_t q = 32; q < j; ++q) t |= glist[q].s == s;
                if (t) e[jj] = E(0);
            }
        };
        Acc tot = 0;
        for (uint32_t r = 0; r < P.nrows; ++r) {
            E e[4];
            masked(r, e);
            VRow<E> row;
            row.compute(e);
            tot += row.tot;
        }
        const Acc x = Tr::draw(U, tot);
        Acc base = 0;
        uint32_t lastp = NONE;
        for (uint32_t r = 0; r < P.nrows; ++r) {
            E e[4];
            masked(r, e);
            VRow<E> row;
            row.compute(e);
            Acc ex = __shfl_up_sync(FULL, row.incl, 1);
            if (lane == 0) ex = 0;
            int jh = -1;
#pragma unroll
            for (int jj = 3; jj >= 0; --jj)
                if (e[jj] > E(0) && base + ex + row.c[jj] > x) jh = jj;
            const unsigned hit = __ballot_sync(FULL, jh >= 0);
            if (hit) {
                const int f = __ffs(hit) - 1;
                return r * VROW + 4 * f + __shfl_sync(FULL, jh, f) - P.head;
            }
            int jl = -1;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
                if (e[jj] > E(0)) jl = jj;
            const unsigned hp = __ballot_sync(FULL, jl >= 0);
            if (hp) {
                const int f = 31 - __clz(hp);
                lastp = r * VROW + 4 * f + __shfl_sync(FULL, jl, f) - P.head;
            }
            base += row.tot;
        }
        return lastp;   // rounding put x past every untaken boundary
    };
    for (uint32_t j = 0; j < k; ++j) {
        uint32_t a = 0;
        uint32_t s;
        if (dk.mode == MIGRATE_UPDATED) {
            s = updated(j, wor_draw(dk, j, 0));
            a = 1;
        } else {
            for (;;) {
                VRegion<E> R = vscan_find(P, C, tab, Tr::draw(wor_draw(dk, j, a), T));
                ++a;
                if (!taken(R.s, j)) { s = R.s; break; }
                if (dk.mode == MIGRATE_BRS) {
                    // (3) fresh draw over the space without [S_s, S_s + b_s); (4)/(5) map back
                    const Acc x2 = Tr::draw(wor_draw(dk, j, a), T - R.b);
                    ++a;
                    const Acc y = x2 < R.lo ? x2 : x2 + R.b;
                    R = vscan_find(P, C, tab, y);
                    if (!taken(R.s, j)) { s = R.s; break; }
                }
                if (a >= a_max) { s = updated(j, wor_draw(dk, j, a_max)); ++a; break; }   // R2
            }
        }
        dk.draws += a;
        if (j < 32) {
            if (static_cast<uint32_t>(lane) == j) mine = s;
        } else if (lane == 0) {
            PickRec pr; pr.s = s; pr.b = 0; pr.lo = 0;
            glist[j] = pr;
        }
        __syncwarp();
    }
    // emit in ascending pool order
    if (k <= 32) {
        const uint32_t sorted = warp_sort_u32(mine);
        if (static_cast<uint32_t>(lane) < k) emit(static_cast<uint32_t>(lane), sorted, P.item(sorted));
    } else {
        for (uint32_t e = 0; e < k; ++e) {
            const uint32_t se = e < 32 ? __shfl_sync(FULL, mine, e) : glist[e].s;
            uint32_t rank = 0;
            for (uint32_t q = lane; q < k; q += 32) {
                const uint32_t sq = q < 32 ? NONE : glist[q].s;
                rank += sq < se;
            }
            rank = __reduce_add_sync(FULL, rank) + __popc(__ballot_sync(FULL, mine < se));
            if (lane == 0) emit(rank, se, P.item(se));
        }
    }
    return k;
}

}  // namespace csaw
