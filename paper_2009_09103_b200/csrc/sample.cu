// sample.cu — traversal sampling: neighbor sampling (degree / uniform bias,
// P:153-154), forest fire and layer sampling.
//
// Level-synchronous driver over ONE batched frontier queue that mixes all
// instances (batched multi-instance sampling): a queue entry is
// (VertexID, InstanceID) with CurrDepth implicit in the level.
// Per level:
//   bound   ub = min(k, deg) per work item (k = NeighborSize, or the burn count)
//   scan    staging offsets
//   select  one warp per pool: EDGEBIAS -> CTPS -> Philox -> ITS -> bitmap/BRS
//           (select.cuh), picks written in canonical (src, dst) order
//   update  UPDATE = visited post-filter (reading R9): candidate keys
//           (instance, vertex) for unvisited picks, LSD radix sort, unique ->
//           next queue sorted by (instance, vertex) (set semantics, R10)
// Finally per-instance offsets are scanned and edges scattered in canonical
// (depth, src, dst) order (R11).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "select.cuh"
#include "vscan.cuh"
#include "util.cuh"

namespace csaw {

constexpr int SEL_WARPS = 8;
constexpr uint64_t SENT = ~0ull;

enum ErrFlag : unsigned { ERR_SEED_RANGE = 1u, ERR_POOL_TOO_BIG = 2u, ERR_K_TOO_BIG = 4u };

struct LevelDesc {                 // device-side view of one level
    const uint32_t* qv;            // queue vertices (sorted within instance)
    const uint64_t* inst_off;      // [n+1] instance segments of the queue
    const uint64_t* eoff;          // [nwork+1] staging offsets
    const uint64_t* rank;          // [total+1] exclusive scan of valid staged entries
    uint64_t* lvlbase;             // [n] edges of this instance in earlier levels
    int layer;                     // work item = instance (layer) or queue entry
};

// ---------------------------------------------------------------- kernels
__global__ void k_init_queue(const uint32_t* __restrict__ seeds, uint64_t n, int64_t V, uint32_t* qv, uint32_t* qi,
                             uint64_t* inst_off, unsigned* err) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n; i += (uint64_t)gridDim.x * blockDim.x) {
        inst_off[i] = i;
        if (i < n) {
            const uint32_t s = seeds[i];
            if (static_cast<int64_t>(s) >= V) atomicOr(err, ERR_SEED_RANGE);
            qv[i] = s;
            qi[i] = static_cast<uint32_t>(i);
        }
    }
}

// Forest-fire burn count: consecutive successes of o0 < theta, truncated at deg (R15).
__device__ __forceinline__ uint32_t ff_burn(uint2 key, uint32_t inst, uint32_t d, uint32_t v, uint32_t deg,
                                            uint64_t theta) {
    uint32_t x = 0;
    while (x < deg) {
        const uint4 o = philox4x32_10(make_uint4(inst, d, v, (PURPOSE_BURN << 28) | x), key);
        if (static_cast<uint64_t>(o.x) < theta) ++x; else break;
    }
    return x;
}

__global__ void k_ns_bound(const int64_t* __restrict__ rp, const uint32_t* __restrict__ qv,
                           const uint32_t* __restrict__ qi, uint64_t nq, int ff, uint32_t fanout, uint64_t theta,
                           uint32_t d, uint32_t base, uint2 key, uint32_t* __restrict__ ub, uint32_t* __restrict__ kq,
                           unsigned* kmax) {
    uint32_t mk = 0;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = qv[q];
        const uint32_t deg = static_cast<uint32_t>(rp[v + 1] - rp[v]);
        const uint32_t k = ff ? ff_burn(key, base + qi[q], d, v, deg, theta) : fanout;
        kq[q] = k;
        ub[q] = min(k, deg);
        if (k < deg) mk = max(mk, k);   // select-all pools (k >= deg) need no pick list / draw index
    }
    mk = __reduce_max_sync(FULL, mk);
    if ((threadIdx.x & 31) == 0 && mk) atomicMax(kmax, mk);
}

struct U32Val {
    const uint32_t* a;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return a[i]; }
};

template <class Pool>
struct StageEmit {
    uint32_t* s_inst;
    uint32_t* s_src;
    uint32_t* s_dst;
    uint64_t e0;
    uint32_t inst;
    uint32_t src;
    __device__ __forceinline__ void operator()(uint32_t rank, uint32_t, uint32_t item) const {
        s_inst[e0 + rank] = inst;
        s_src[e0 + rank] = src;
        s_dst[e0 + rank] = item;
    }
};

struct SelArgs {
    const int64_t* __restrict__ rp;
    const uint32_t* __restrict__ col;
    const uint32_t* __restrict__ deg;
    const uint32_t* __restrict__ qv;
    const uint32_t* __restrict__ qi;
    uint64_t nq;
    const uint32_t* __restrict__ kq;
    const uint32_t* __restrict__ ub;
    const uint64_t* __restrict__ eoff;
    uint32_t* s_inst;
    uint32_t* s_src;
    uint32_t* s_dst;
    uint32_t d;
    uint32_t base;
    uint2 key;
    uint32_t a_max;
    PickRec* glist;
    uint32_t kmax;
    unsigned long long* counters;   // [0] scanned, [1] pools, [2] cache probes, [3] draws
    const uint64_t* __restrict__ cps;    // static-bias CTPS cache (nullptr if not built)
    const uint32_t* __restrict__ npos;
    const uint64_t* __restrict__ bt;
    const uint64_t* __restrict__ bt_off;
    uint32_t mode;                   // collision migration (MIGRATE_*)
    const uint32_t* __restrict__ qidx;   // OOM: queue entries of one partition (nullptr = all nq entries)
    uint64_t nidx;
    const uint64_t* __restrict__ ccache;  // chunk-total cache (degree pools), optional
    WixPtrs wx;                           // vertex heads (cached degree pools), optional
    const float* __restrict__ w = nullptr;   // edge weights (kMode 3)
};

// Neighbor sampling / forest fire: one warp per queue entry.
// kMode: 0 = uniform (closed form), 1 = degree (scanned CTPS), 2 = degree (cached CTPS),
//        3 = edge weights (float CTPS over the weight stream, vscan.cuh; R28)
template <int kMode>
__global__ void __launch_bounds__(SEL_WARPS * 32, 3) k_ns_select(SelArgs a) {
    __shared__ uint64_t tab_all[SEL_WARPS][TAB];
    __shared__ uint32_t bm_all[SEL_WARPS][BM_WORDS];
    const int wib = threadIdx.x >> 5;
    uint64_t* tab = tab_all[wib];
    uint32_t* bm = bm_all[wib];
    const int lane = lane_id();
    PickRec* gl = a.glist ? a.glist + global_warp_id() * a.kmax : nullptr;
    unsigned long long scanned = 0, pools = 0, probes = 0, draws = 0;
    const uint64_t nwork = a.qidx ? a.nidx : a.nq;
    for (uint64_t jq = global_warp_id(); jq < nwork; jq += total_warps()) {
        const uint64_t q = a.qidx ? a.qidx[jq] : jq;
        const uint32_t v = a.qv[q];
        const uint32_t inst = a.qi[q];
        const int64_t b0 = __ldg(a.rp + v);
        const uint32_t n = static_cast<uint32_t>(__ldg(a.rp + v + 1) - b0);
        const uint32_t k = a.kq[q];
        const uint64_t e0 = a.eoff[q];
        const uint32_t ub = a.ub[q];
        DrawKey dk{a.key, a.base + inst, a.d, v, a.mode, 0};
        StageEmit<int> emit{a.s_inst, a.s_src, a.s_dst, e0, inst, v};
        uint32_t cnt = 0;
        if (n > 0 && k > 0) {
            if constexpr (kMode == 2) {
                CachedDegreePool P{a.col, a.cps, static_cast<uint64_t>(b0), n, __ldg(a.npos + v), 0, a.bt,
                                   a.wx.head ? 0 : __ldg(a.bt_off + v)};
                P.wx = a.wx;
                P.vid = v;
                const Ctps C = build_ctps(P, tab);
                cnt = select_wor(P, C, tab, bm, k, dk, a.a_max, gl, emit);
                probes += P.probes;
            } else if constexpr (kMode == 1) {
                DegreePool P{a.col, a.deg, static_cast<uint64_t>(b0), n, a.ccache};
                const Ctps C = build_ctps(P, tab);
                cnt = select_wor(P, C, tab, bm, k, dk, a.a_max, gl, emit);
                scanned += (a.ccache && C.m) ? 32u * C.m : n;   // chunk cache: ~one chunk rescanned per pick
            } else if constexpr (kMode == 3) {
                VPool<float> P;
                P.init(a.w, a.col, static_cast<uint64_t>(b0), n);
                double* ftab = reinterpret_cast<double*>(tab);
                const VCtps<float> C = vscan_build<float, 1>(P, ftab, nullptr, 0, [] {});
                cnt = vscan_select_wor(P, C, ftab, k, dk, a.a_max, gl, emit);
                scanned += n;
            } else {
                UniformPool P{a.col, static_cast<uint64_t>(b0), n};
                const Ctps C = build_ctps(P, tab);
                cnt = select_wor(P, C, tab, bm, k, dk, a.a_max, gl, emit);
            }
            ++pools;
            draws += dk.draws;
        }
        for (uint32_t r = cnt + lane; r < ub; r += 32) {
            a.s_inst[e0 + r] = inst;
            a.s_src[e0 + r] = v;
            a.s_dst[e0 + r] = NONE;
        }
    }
    if (lane == 0) {
        if (scanned) atomicAdd(a.counters + 0, scanned);
        if (pools) atomicAdd(a.counters + 1, pools);
        if (probes) atomicAdd(a.counters + 2, probes);
        if (draws) atomicAdd(a.counters + 3, draws);
    }
}

// ---------------------------------------------------------------- layer sampling
// Pool = multiset union of N(v) over the instance's sorted frontier, in that
// order (reading R14); EDGEBIAS = deg(u).  seg_pref[j] = sum of frontier
// degrees before segment j (relative to the instance).
template <bool kCache>
struct LayerPoolT {
    static constexpr bool kClosedForm = false;
    static constexpr bool kCached = kCache;
    const int64_t* __restrict__ rp;
    const uint32_t* __restrict__ col;
    const uint32_t* __restrict__ deg;
    const uint64_t* __restrict__ cps;    // static-bias CTPS cache (kCache)
    const uint32_t* __restrict__ npos;   // positive-bias neighbours per row (kCache)
    const uint64_t* __restrict__ bt;     // B-tree index over cps (kCache)
    const uint64_t* __restrict__ bt_off;
    WixPtrs wx{};                        // vertex heads (optional; kCache)
    const uint32_t* fv;                  // frontier vertices of the instance (global or shared)
    const uint64_t* pref;                // exclusive prefix of frontier degrees (global or shared)
    uint64_t pbase;                      // pref at the instance's first segment
    uint32_t nf;                         // frontier size
    uint32_t n;                          // pool size
    uint32_t probes;
    // per-lane cursor
    uint32_t seg;
    uint64_t seg_lo, seg_hi;             // pool range of segment seg
    int64_t seg_row;                     // rp[fv[seg]]

    __device__ __forceinline__ uint32_t find_seg(uint64_t i) const {   // last j with pref_rel[j] <= i
        uint32_t lo = 0, hi = nf;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pref[mid] - pbase <= i) lo = mid; else hi = mid;
        }
        return lo;
    }
    __device__ __forceinline__ void set_seg(uint32_t j) {
        seg = j;
        seg_lo = pref[j] - pbase;
        seg_hi = (j + 1 < nf) ? pref[j + 1] - pbase : n;
        seg_row = __ldg(rp + fv[j]);
    }
    __device__ __forceinline__ void seek(uint32_t row0) {
        const uint64_t i = static_cast<uint64_t>(row0) * 32 + lane_id();
        set_seg(i < n ? find_seg(i) : nf - 1);
    }
    template <int NR>
    __device__ __forceinline__ void load_rows(uint32_t row0, uint32_t (&key)[NR], uint32_t (&b)[NR]) {
        const int lane = lane_id();
        int64_t eidx[NR], rs[NR];
#pragma unroll
        for (int u = 0; u < NR; ++u) {
            const uint64_t i = static_cast<uint64_t>(row0 + u) * 32 + lane;
            eidx[u] = -1;
            rs[u] = 0;
            if (i < n) {
                while (i >= seg_hi) set_seg(seg + 1);
                eidx[u] = seg_row + static_cast<int64_t>(i - seg_lo);
                rs[u] = seg_row;
                key[u] = __ldg(col + eidx[u]);
            } else {
                key[u] = NONE;
            }
        }
#pragma unroll
        for (int u = 0; u < NR; ++u) {
            if constexpr (kCache) {
                b[u] = 0;
                if (eidx[u] >= 0) {
                    const int64_t e = eidx[u];
                    b[u] = static_cast<uint32_t>(__ldg(cps + e) - (e == rs[u] ? 0 : __ldg(cps + e - 1)));
                }
            } else {
                b[u] = (key[u] != NONE) ? __ldg(deg + key[u]) : 0u;
            }
        }
    }
    __device__ __forceinline__ uint32_t item(uint32_t i) const {
        const uint32_t j = find_seg(i);
        const uint32_t v = fv[j];
        return __ldg(col + __ldg(rp + v) + (i - (pref[j] - pbase)));
    }
    __device__ __forceinline__ uint32_t src_of(uint32_t i) const { return fv[find_seg(i)]; }

    // ---- cached CTPS of the union pool: segment j contributes [O_j, O_j + T_j)
    __device__ __forceinline__ uint64_t seg_total(uint32_t j) const {
        const uint32_t v = fv[j];
        const int64_t a = __ldg(rp + v), b = __ldg(rp + v + 1);
        return b > a ? __ldg(cps + b - 1) : 0;
    }
    __device__ __forceinline__ uint64_t total() const {
        uint64_t t = 0;
        for (uint32_t j0 = 0; j0 < nf; j0 += 32) {
            const uint32_t j = j0 + lane_id();
            t += warp_sum(j < nf ? seg_total(j) : 0);
        }
        return t;
    }
    __device__ __forceinline__ uint32_t npos_count() const {
        uint32_t t = 0;
        for (uint32_t j0 = 0; j0 < nf; j0 += 32) {
            const uint32_t j = j0 + lane_id();
            t += __reduce_add_sync(FULL, j < nf ? __ldg(npos + fv[j]) : 0u);
        }
        return t;
    }
    __device__ __forceinline__ Region search(uint64_t x) {   // x warp-uniform
        uint64_t base = 0, O = 0;
        uint32_t js = 0;
        for (uint32_t j0 = 0; j0 < nf; j0 += 32) {
            const uint32_t j = j0 + lane_id();
            const uint64_t tj = j < nf ? seg_total(j) : 0;
            const uint64_t incl = warp_incl_scan(tj) + base;
            const unsigned hit = __ballot_sync(FULL, j < nf && incl > x);
            if (hit) {
                const int f = __ffs(hit) - 1;
                js = j0 + f;
                O = __shfl_sync(FULL, incl - tj, f);
                break;
            }
            base = __shfl_sync(FULL, incl, 31);
        }
        const uint32_t v = fv[js];
        if (wx.head) {   // vertex head -> (node) -> leaf; S < 2^32 for every row
            uint32_t s, lo, b, it, nb;
            wix_head_search<128>(wx.head, wx.c32, wx.col, wx.inn, v, static_cast<uint32_t>(x - O), s, lo, b, it, nb);
            probes += nb / 8;   // in 8 B cache-entry units (statistics)
            Region r;
            r.s = static_cast<uint32_t>((pref[js] - pbase) + s);
            r.lo = O + lo;
            r.b = b;
            r.item = it;
            return r;
        }
        const int64_t ra = __ldg(rp + v), rb = __ldg(rp + v + 1);
        CpsTree t{cps, bt, col, static_cast<uint64_t>(ra), static_cast<uint32_t>(rb - ra), __ldg(bt_off + v)};
        uint64_t xl = x - O, T = 0, e = 0, lo = 0, hi = 0;
        uint32_t item = NONE;
        t.template search<false>(0, xl, T, e, lo, hi, item, probes);
        Region r;
        r.s = static_cast<uint32_t>((pref[js] - pbase) + (e - static_cast<uint64_t>(ra)));
        r.lo = O + lo;
        r.b = static_cast<uint32_t>(hi - lo);
        r.item = item;
        return r;
    }
};
using LayerPool = LayerPoolT<false>;

template <class LP>
struct LayerEmit {
    const LP* P;
    uint32_t* s_inst;
    uint32_t* s_src;
    uint32_t* s_dst;
    uint64_t e0;
    uint32_t inst;
    __device__ __forceinline__ void operator()(uint32_t rank, uint32_t s, uint32_t item) const {
        s_inst[e0 + rank] = inst;
        s_src[e0 + rank] = P->src_of(s);
        s_dst[e0 + rank] = item;
    }
};

struct DegOfQueue {
    const int64_t* rp;
    const uint32_t* qv;
    __device__ __forceinline__ uint64_t operator()(uint64_t q) const {
        const uint32_t v = qv[q];
        return static_cast<uint64_t>(rp[v + 1] - rp[v]);
    }
};

__global__ void k_layer_bound(const uint64_t* __restrict__ inst_off, const uint64_t* __restrict__ qpref, uint64_t n,
                              uint32_t fanout, uint32_t* __restrict__ ub, unsigned* err, unsigned* kmax) {
    uint32_t mk = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t P = qpref[inst_off[i + 1]] - qpref[inst_off[i]];
        if (P >= static_cast<uint64_t>(NONE) - 64) atomicOr(err, ERR_POOL_TOO_BIG);
        ub[i] = static_cast<uint32_t>(min(static_cast<uint64_t>(fanout), P));
        mk = max(mk, ub[i]);
    }
    mk = __reduce_max_sync(FULL, mk);
    if ((threadIdx.x & 31) == 0 && mk) atomicMax(kmax, mk);
}

struct LayerArgs {
    const int64_t* __restrict__ rp;
    const uint32_t* __restrict__ col;
    const uint32_t* __restrict__ deg;
    const uint32_t* __restrict__ qv;
    const uint64_t* __restrict__ inst_off;
    const uint64_t* __restrict__ qpref;
    uint64_t n;
    uint32_t fanout;
    const uint32_t* __restrict__ ub;
    const uint64_t* __restrict__ eoff;
    uint32_t* s_inst;
    uint32_t* s_src;
    uint32_t* s_dst;
    uint32_t d;
    uint32_t base;
    uint2 key;
    uint32_t a_max;
    PickRec* glist;
    uint32_t kmax;
    unsigned long long* counters;
    const uint64_t* __restrict__ cps;
    const uint32_t* __restrict__ npos;
    const uint64_t* __restrict__ bt;
    const uint64_t* __restrict__ bt_off;
    uint32_t mode;
    WixPtrs wx;                          // vertex heads, optional
};

// one warp per instance (its layer pool); kCache: union CTPS from the static-bias cache
template <bool kCache>
__global__ void __launch_bounds__(SEL_WARPS * 32, 3) k_layer_select(LayerArgs a) {
    __shared__ uint64_t tab_all[SEL_WARPS][TAB];
    __shared__ uint32_t bm_all[SEL_WARPS][BM_WORDS];
    const int wib = threadIdx.x >> 5;
    uint64_t* tab = tab_all[wib];
    uint32_t* bm = bm_all[wib];
    const int lane = lane_id();
    PickRec* gl = a.glist ? a.glist + global_warp_id() * a.kmax : nullptr;
    unsigned long long scanned = 0, pools = 0, probes = 0, draws = 0;
    for (uint64_t i = global_warp_id(); i < a.n; i += total_warps()) {
        const uint64_t qb = a.inst_off[i], qe = a.inst_off[i + 1];
        const uint64_t e0 = a.eoff[i];
        const uint32_t ub = a.ub[i];
        uint32_t cnt = 0;
        if (qe > qb && ub > 0) {
            LayerPoolT<kCache> P;
            P.rp = a.rp; P.col = a.col; P.deg = a.deg; P.cps = a.cps; P.npos = a.npos; P.probes = 0; P.wx = a.wx;
            P.bt = a.bt; P.bt_off = a.bt_off;
            P.fv = a.qv + qb;
            P.pref = a.qpref + qb;
            P.pbase = a.qpref[qb];
            P.nf = static_cast<uint32_t>(qe - qb);
            P.n = static_cast<uint32_t>(a.qpref[qe] - P.pbase);
            DrawKey dk{a.key, a.base + static_cast<uint32_t>(i), a.d, NONE, a.mode, 0};
            LayerEmit<LayerPoolT<kCache>> emit{&P, a.s_inst, a.s_src, a.s_dst, e0, static_cast<uint32_t>(i)};
            const Ctps C = build_ctps(P, tab);
            cnt = select_wor(P, C, tab, bm, a.fanout, dk, a.a_max, gl, emit);
            if (!kCache) scanned += P.n;
            probes += P.probes;
            ++pools;
            draws += dk.draws;
        }
        for (uint32_t r = cnt + lane; r < ub; r += 32) {
            a.s_inst[e0 + r] = static_cast<uint32_t>(i);
            a.s_src[e0 + r] = NONE;
            a.s_dst[e0 + r] = NONE;
        }
    }
    if (lane == 0) {
        if (scanned) atomicAdd(a.counters + 0, scanned);
        if (pools) atomicAdd(a.counters + 1, pools);
        if (probes) atomicAdd(a.counters + 2, probes);
        if (draws) atomicAdd(a.counters + 3, draws);
    }
}

// ---------------------------------------------------------------- UPDATE: next frontier
struct VisitedArgs {
    const uint32_t* seeds;
    const LevelDesc* levels;   // levels[1..l] have queues; level 0 = seeds
    int nlev;                  // number of queue levels to check beyond the seed (1..l)
};

__device__ __forceinline__ bool in_sorted(const uint32_t* a, uint64_t lo, uint64_t hi, uint32_t x) {
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        const uint32_t y = a[mid];
        if (y == x) return true;
        if (y < x) lo = mid + 1; else hi = mid;
    }
    return false;
}

__global__ void k_cand(const uint32_t* __restrict__ s_inst, const uint32_t* __restrict__ s_dst, uint64_t total,
                       VisitedArgs va, int vbits, uint64_t* __restrict__ keys) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = s_dst[e];
        uint64_t key = SENT;
        if (u != NONE) {
            const uint32_t i = s_inst[e];
            bool vis = va.seeds[i] == u;
            for (int l = 1; l <= va.nlev && !vis; ++l) {
                const LevelDesc& L = va.levels[l];
                vis = in_sorted(L.qv, L.inst_off[i], L.inst_off[i + 1], u);
            }
            if (!vis) key = (static_cast<uint64_t>(i) << vbits) | u;
        }
        keys[e] = key;
    }
}

struct UniqueFlag {
    const uint64_t* k;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
        const uint64_t x = k[i];
        return (x != SENT && (i == 0 || x != k[i - 1])) ? 1u : 0u;
    }
};

struct CompactQueue {
    const uint64_t* k;
    uint32_t* qv;
    uint32_t* qi;
    uint64_t* count;
    int vbits;
    __device__ __forceinline__ void operator()(uint64_t i, uint64_t e, uint64_t v) const {
        if (v) {
            const uint64_t x = k[i];
            qv[e] = static_cast<uint32_t>(x & ((1ull << vbits) - 1));
            qi[e] = static_cast<uint32_t>(x >> vbits);
        }
    }
    __device__ __forceinline__ void total(uint64_t, uint64_t t) const { *count = t; }
};

__global__ void k_inst_off(const uint32_t* __restrict__ qi, uint64_t nq, uint64_t n, uint64_t* __restrict__ off) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = nq;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (qi[mid] < i) lo = mid + 1; else hi = mid;
        }
        off[i] = lo;
    }
}

// ---- segmented UPDATE (common case): one warp per instance sorts + dedups its own
// candidates in shared memory (they are contiguous in the staging array), applies
// the visited post-filter, and writes its next-frontier segment; a scan of the
// per-instance counts gives the next queue's instance offsets directly.
constexpr uint32_t FSEG = 1024;   // max staged picks per instance handled by the segmented path
constexpr int FSEG_WARPS = 4;

__device__ __forceinline__ uint64_t stage_begin_l(const uint64_t* eoff, const uint64_t* inst_off, int layer, uint64_t i) {
    return layer ? eoff[i] : eoff[inst_off[i]];
}

__global__ void k_segmax(const uint64_t* __restrict__ eoff, const uint64_t* __restrict__ inst_off, int layer,
                         uint64_t n, unsigned* segmax) {
    uint32_t mk = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = stage_begin_l(eoff, inst_off, layer, i + 1) - stage_begin_l(eoff, inst_off, layer, i);
        mk = max(mk, static_cast<uint32_t>(min(c, static_cast<uint64_t>(0xFFFFFFFFu))));
    }
    mk = __reduce_max_sync(FULL, mk);
    if ((threadIdx.x & 31) == 0 && mk) atomicMax(segmax, mk);
}

__global__ void __launch_bounds__(FSEG_WARPS * 32) k_frontier_seg(const uint64_t* __restrict__ eoff,
                                                                  const uint64_t* __restrict__ inst_off, int layer,
                                                                  const uint32_t* __restrict__ s_dst, VisitedArgs va,
                                                                  uint64_t n, uint32_t* __restrict__ tmp,
                                                                  uint64_t* __restrict__ cnt) {
    __shared__ uint32_t buf_all[FSEG_WARPS][FSEG];
    uint32_t* buf = buf_all[threadIdx.x >> 5];
    const int lane = lane_id();
    for (uint64_t i = global_warp_id(); i < n; i += total_warps()) {
        const uint64_t sb = stage_begin_l(eoff, inst_off, layer, i);
        const uint32_t c = static_cast<uint32_t>(stage_begin_l(eoff, inst_off, layer, i + 1) - sb);
        uint32_t P = 32;
        while (P < c) P <<= 1;
        for (uint32_t j = lane; j < P; j += 32) {
            uint32_t u = NONE;
            if (j < c) {
                u = s_dst[sb + j];
                if (u != NONE) {   // UPDATE: drop vertices this instance already visited (R9)
                    bool vis = va.seeds[i] == u;
                    for (int l = 1; l <= va.nlev && !vis; ++l) {
                        const LevelDesc& L = va.levels[l];
                        vis = in_sorted(L.qv, L.inst_off[i], L.inst_off[i + 1], u);
                    }
                    if (vis) u = NONE;
                }
            }
            buf[j] = u;
        }
        __syncwarp();
        // bitonic sort of buf[0, P) ascending (NONE sorts last)
        for (uint32_t k = 2; k <= P; k <<= 1) {
            for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
                for (uint32_t idx = lane; idx < P; idx += 32) {
                    const uint32_t pr = idx ^ jj;
                    if (pr > idx) {
                        const uint32_t a = buf[idx], b = buf[pr];
                        const bool up = (idx & k) == 0;
                        if ((a > b) == up) { buf[idx] = b; buf[pr] = a; }
                    }
                }
                __syncwarp();
            }
        }
        // unique, compacted into tmp[sb ...) (set semantics, R10)
        uint32_t w = 0;
        for (uint32_t j0 = 0; j0 < c; j0 += 32) {
            const uint32_t j = j0 + lane;
            const uint32_t u = j < c ? buf[j] : NONE;
            const bool keep = u != NONE && (j == 0 || buf[j - 1] != u);
            const unsigned bal = __ballot_sync(FULL, keep);
            if (keep) tmp[sb + w + __popc(bal & lanemask_lt())] = u;
            w += __popc(bal);
        }
        if (lane == 0) cnt[i] = w;
        __syncwarp();
    }
}

__global__ void k_frontier_compact(const uint64_t* __restrict__ eoff, const uint64_t* __restrict__ inst_off, int layer,
                                   const uint32_t* __restrict__ tmp, const uint64_t* __restrict__ noff, uint64_t n,
                                   uint32_t* __restrict__ nqv, uint32_t* __restrict__ nqi) {
    const int lane = lane_id();
    for (uint64_t i = global_warp_id(); i < n; i += total_warps()) {
        const uint64_t sb = stage_begin_l(eoff, inst_off, layer, i);
        const uint64_t o = noff[i], c = noff[i + 1] - o;
        for (uint64_t j = lane; j < c; j += 32) {
            nqv[o + j] = tmp[sb + j];
            nqi[o + j] = static_cast<uint32_t>(i);
        }
    }
}

struct ValidVal {
    const uint32_t* s_dst;
    __device__ __forceinline__ uint64_t operator()(uint64_t e) const { return s_dst[e] != NONE ? 1u : 0u; }
};

// ---------------------------------------------------------------- final assembly
__device__ __forceinline__ uint64_t stage_begin(const LevelDesc& L, uint64_t i) {
    return L.layer ? L.eoff[i] : L.eoff[L.inst_off[i]];
}

__global__ void k_counts(const LevelDesc* __restrict__ levels, int nlev, uint64_t n, uint64_t* __restrict__ tot) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t run = 0;
        for (int l = 0; l < nlev; ++l) {
            const LevelDesc& L = levels[l];
            const uint64_t c = L.rank[stage_begin(L, i + 1)] - L.rank[stage_begin(L, i)];
            L.lvlbase[i] = run;
            run += c;
        }
        tot[i] = run;
    }
}

struct U64Val {
    const uint64_t* a;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return a[i]; }
};

__global__ void k_write(LevelDesc L, int depth1, const uint32_t* __restrict__ s_inst, const uint32_t* __restrict__ s_src,
                        const uint32_t* __restrict__ s_dst, uint64_t total, const uint64_t* __restrict__ offsets,
                        uint32_t* __restrict__ src, uint32_t* __restrict__ dst, uint8_t* __restrict__ dep) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = s_dst[e];
        if (u == NONE) continue;
        const uint32_t i = s_inst[e];
        const uint64_t pos = offsets[i] + L.lvlbase[i] + L.rank[e] - L.rank[stage_begin(L, i)];
        src[pos] = s_src[e];
        dst[pos] = u;
        dep[pos] = static_cast<uint8_t>(depth1);
    }
}

// ---------------------------------------------------------------- OOM: partition-grouped levels
// Batched multi-instance sampling in the out-of-memory mode (§5.2-5.3):
// a level's queue (all instances mixed) is grouped by the partition owning each
// frontier vertex; partitions are made resident busiest-first and one select
// kernel per resident partition processes its entries (CTAs ~ its count).  Levels
// run in order, so the visited filter sees complete earlier levels (R22).
struct OwnerP {
    uint64_t base, rem;
    __device__ __forceinline__ uint32_t operator()(uint32_t v) const {
        const uint64_t big = rem * (base + 1);
        if (v < big) return static_cast<uint32_t>(v / (base + 1));
        return static_cast<uint32_t>(rem + (v - big) / base);
    }
};

__global__ void k_part_count(const uint32_t* __restrict__ qv, uint64_t nq, OwnerP own, uint32_t* __restrict__ cnt) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + own(qv[q]), 1u);
}

__global__ void k_part_scatter(const uint32_t* __restrict__ qv, uint64_t nq, OwnerP own, uint32_t* __restrict__ fill,
                               uint32_t* __restrict__ idx) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t pos = atomicAdd(fill + own(qv[q]), 1u);   // fill[p] starts at partition p's offset
        idx[pos] = static_cast<uint32_t>(q);
    }
}

// ---------------------------------------------------------------- fused per-instance sampler
// For small per-instance frontiers (the paper's NeighborSize = Depth = 2 setups,
// P:972-974) the whole traversal of one instance runs in ONE warp: frontier,
// next frontier and visited set live in shared memory, each level's pools are
// selected in frontier order, and the edges go to a per-instance staging row.
// One launch instead of ~15 per level and no host round trip between levels;
// the results are identical to the level-synchronous batched driver because
// every draw is keyed by (instance, depth, vertex) (R7).  Anything that does not
// fit (frontier > F_CAP, visited > VIS_CAP, more staged edges than ecap, or a
// pool needing > 32 picks) raises the overflow flag and the host reruns the call
// with the batched driver.
#ifndef FUSED_WARPS_N
#define FUSED_WARPS_N 4
#endif
constexpr int FUSED_WARPS = FUSED_WARPS_N;   // warps (instances in flight) per block
#ifndef FUSED_MINB
#define FUSED_MINB 4
#endif
#ifndef FUSED_FF_MINB
#define FUSED_FF_MINB 8
#endif
constexpr uint32_t F_CAP = 256;
constexpr uint32_t VIS_CAP = 512;
// layer sampling: a level's frontier is its fanout distinct picks (<= 32), so the layer kernels
// keep 64-entry frontiers and a 256-entry visited list -- 24 KB of shared memory per 4-warp
// block instead of 36 KB, and 64 registers: 8 blocks (32 warps) per SM instead of 6
// (A/B cfg4 layer: 0.109 vs 0.119 ms per step); larger visited sets overflow to the batched driver
constexpr uint32_t F_CAP_LAYER = 64;
constexpr uint32_t VIS_CAP_LAYER = 256;

struct FusedArgs {
    const int64_t* __restrict__ rp;
    const uint32_t* __restrict__ col;
    const uint32_t* __restrict__ deg;
    const uint64_t* __restrict__ cps;
    const uint32_t* __restrict__ npos;
    const uint64_t* __restrict__ bt;
    const uint64_t* __restrict__ bt_off;
    const uint32_t* __restrict__ seeds;
    uint64_t n;
    int32_t depth;
    int32_t fanout[16];                   // per level (kernel parameter: no copy per call)
    uint64_t theta;                       // forest fire
    uint32_t base;
    uint2 key;
    uint32_t a_max;
    uint32_t ecap;                        // staged edges per instance
    uint32_t* __restrict__ s_src;         // [n][ecap]
    uint32_t* __restrict__ s_dst;
    uint8_t* __restrict__ s_dep;
    uint64_t* __restrict__ cnt;           // [n]
    unsigned* overflow;                   // bit 0: fall back to the batched driver; bit 1: seed out of range
    unsigned long long* counters;
    int64_t V;
    uint32_t mode;
    // epilogue (last block to finish): offsets scan + the host report
    uint64_t* offs;                       // [n + 1] exclusive prefix of cnt (caller's offsets)
    uint64_t* offs_host;                  // optional pinned host copy (device-mapped), written alongside
    unsigned* done;                       // block ticket (zeroed with the counters each call)
    uint64_t* report;                     // pinned host mailbox: flags, total, counters[0..3]
    const uint64_t* __restrict__ ccache;  // chunk-total cache (degree pools), optional
    WixPtrs wx;                           // vertex heads (cached degree / layer pools), optional
    const float* __restrict__ w = nullptr;   // edge weights (kMode 6)
};

// Run by the last block of k_sample_fused to finish (ticket): the per-instance edge
// offsets (exclusive prefix of cnt, one block) and the call's report written straight
// into pinned host memory -- two launches less per call than a separate scan + report.
template <int NT>
__device__ void fused_epilogue(const FusedArgs& a) {
    __shared__ unsigned last;
    __shared__ uint64_t wsum[NT / 32];
    __shared__ uint64_t total;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(a.done, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const uint64_t n = a.n;
    const uint64_t per = (n + NT - 1) / NT;
    const uint64_t b0 = min(n, threadIdx.x * per), b1 = min(n, b0 + per);
    // 8 independent loads in flight per thread (the counts sit in L2)
    uint64_t s = 0;
    for (uint64_t i0 = b0; i0 < b1; i0 += 8) {
        uint64_t c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = i0 + u < b1 ? __ldcg(a.cnt + i0 + u) : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) s += c[u];
    }
    uint64_t run = block_excl_scan<NT>(s, wsum, &total);
    // pinned host offsets only for a call that succeeds here: a bad seed (bit 1) or a fallback
    // to the batched driver (bit 0) leaves the caller's host buffer untouched
    uint64_t* const offs_host = *reinterpret_cast<volatile unsigned*>(a.overflow) ? nullptr : a.offs_host;
    for (uint64_t i0 = b0; i0 < b1; i0 += 8) {
        uint64_t c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = i0 + u < b1 ? __ldcg(a.cnt + i0 + u) : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (i0 + u < b1) {
                a.offs[i0 + u] = run;
                if (offs_host) offs_host[i0 + u] = run;
            }
            run += c[u];
        }
    }
    if (threadIdx.x == 0) {
        a.offs[n] = total;
        if (offs_host) offs_host[n] = total;
        a.report[0] = *reinterpret_cast<volatile unsigned*>(a.overflow);
        a.report[1] = total;
        for (int k = 0; k < 4; ++k) a.report[2 + k] = reinterpret_cast<volatile unsigned long long*>(a.counters)[k];
        __threadfence_system();
    }
}

struct FusedEmit {
    uint32_t* s_src;
    uint32_t* s_dst;
    uint8_t* s_dep;
    uint64_t e0;
    uint32_t src;
    uint8_t d1;
    __device__ __forceinline__ void operator()(uint32_t rank, uint32_t, uint32_t item) const {
        s_src[e0 + rank] = src;
        s_dst[e0 + rank] = item;
        s_dep[e0 + rank] = d1;
    }
};

template <class LP>
struct FusedLayerEmit {
    const LP* P;
    uint32_t* s_src;
    uint32_t* s_dst;
    uint8_t* s_dep;
    uint64_t e0;
    uint8_t d1;
    __device__ __forceinline__ void operator()(uint32_t rank, uint32_t s, uint32_t item) const {
        s_src[e0 + rank] = P->src_of(s);
        s_dst[e0 + rank] = item;
        s_dep[e0 + rank] = d1;
    }
};

// kMode: 0 uniform NS, 1 degree NS (scan), 2 degree NS (cache), 3 forest fire,
//        4 layer (scan), 5 layer (cache), 6 edge-weight NS (float CTPS, vscan.cuh; R28)
template <int kMode>
// blocks / SM: forest fire (no layer prefix table, 7 KB smem per warp) 8, layer 6 (smem-bound), NS 4
__global__ void __launch_bounds__(FUSED_WARPS * 32, (kMode == 3 ? FUSED_FF_MINB : (kMode == 4 || kMode == 5) ? 8 : FUSED_MINB) * 4 / FUSED_WARPS)
    k_sample_fused(FusedArgs a) {
    __shared__ uint64_t tab_all[FUSED_WARPS][TAB];
    __shared__ uint32_t bm_all[FUSED_WARPS][BM_WORDS];
    constexpr uint32_t kF = (kMode == 4 || kMode == 5) ? F_CAP_LAYER : F_CAP;
    constexpr uint32_t kVIS = (kMode == 4 || kMode == 5) ? VIS_CAP_LAYER : VIS_CAP;
    __shared__ uint32_t F_all[FUSED_WARPS][kF];
    __shared__ uint32_t NX_all[FUSED_WARPS][kF];
    __shared__ uint32_t VIS_all[FUSED_WARPS][kVIS];
    __shared__ uint64_t PF_all[FUSED_WARPS][(kMode == 4 || kMode == 5) ? kF : 1];   // layer pools only
    const int wib = threadIdx.x >> 5;
    uint64_t* tab = tab_all[wib];
    uint32_t* bm = bm_all[wib];
    uint32_t* F = F_all[wib];
    uint32_t* NX = NX_all[wib];
    uint32_t* VIS = VIS_all[wib];
    uint64_t* PF = PF_all[wib];
    const int lane = lane_id();
    constexpr bool kLayer = kMode == 4 || kMode == 5;
    unsigned long long scanned = 0, pools = 0, probes = 0, draws = 0;
    for (uint64_t i = global_warp_id(); i < a.n; i += total_warps()) {
        const uint32_t inst = a.base + static_cast<uint32_t>(i);
        const uint32_t seed = a.seeds[i];
        const uint64_t e_base = i * a.ecap;
        if (static_cast<int64_t>(seed) >= a.V) {
            if (lane == 0) { atomicOr(a.overflow, 2u); a.cnt[i] = 0; }
            continue;
        }
        if (lane == 0) { F[0] = seed; VIS[0] = seed; }
        __syncwarp();
        uint32_t nf = 1, nv = 1;
        uint32_t ec = 0;
        bool ovf = false;
        for (int32_t d = 0; d < a.depth && nf > 0 && !ovf; ++d) {
            uint32_t nnx = 0;
            const uint32_t ec0 = ec;
            if constexpr (kLayer) {
                // union pool over the sorted frontier: exclusive degree prefix in PF
                uint64_t carry = 0;
                for (uint32_t j0 = 0; j0 < nf; j0 += 32) {
                    const uint32_t j = j0 + lane;
                    const uint64_t dj = j < nf ? static_cast<uint64_t>(__ldg(a.rp + F[j] + 1) - __ldg(a.rp + F[j])) : 0;
                    const uint64_t incl = warp_incl_scan(dj) + carry;
                    if (j < nf) PF[j] = incl - dj;
                    carry = __shfl_sync(FULL, incl, 31);
                }
                __syncwarp();
                const uint32_t k = static_cast<uint32_t>(a.fanout[d]);
                if (carry >= static_cast<uint64_t>(NONE) - 64 || k > 32) { ovf = true; break; }
                const uint32_t pn = static_cast<uint32_t>(carry);
                if (pn > 0 && k > 0) {
                    if (ec + min(k, pn) > a.ecap) { ovf = true; break; }
                    LayerPoolT<kMode == 5> P;
                    P.rp = a.rp; P.col = a.col; P.deg = a.deg; P.cps = a.cps; P.npos = a.npos; P.probes = 0; P.wx = a.wx;
                    P.bt = a.bt; P.bt_off = a.bt_off;
                    P.fv = F; P.pref = PF; P.pbase = 0; P.nf = nf; P.n = pn;
                    DrawKey dk{a.key, inst, static_cast<uint32_t>(d), NONE, a.mode, 0};
                    FusedLayerEmit<LayerPoolT<kMode == 5>> emit{&P, a.s_src, a.s_dst, a.s_dep, e_base + ec,
                                                                 static_cast<uint8_t>(d + 1)};
                    const Ctps C = build_ctps(P, tab);
                    ec += select_wor(P, C, tab, bm, k, dk, a.a_max, nullptr, emit);
                    if (kMode == 4) scanned += pn;
                    probes += P.probes;
                    ++pools;
            draws += dk.draws;
                }
            } else {
                for (uint32_t fj = 0; fj < nf && !ovf; ++fj) {
                    const uint32_t v = F[fj];
                    const int64_t b0 = __ldg(a.rp + v);
                    const uint32_t nd = static_cast<uint32_t>(__ldg(a.rp + v + 1) - b0);
                    uint32_t k;
                    if constexpr (kMode == 3) k = ff_burn(a.key, inst, static_cast<uint32_t>(d), v, nd, a.theta);
                    else k = static_cast<uint32_t>(a.fanout[d]);
                    if (nd == 0 || k == 0) continue;
                    if (k > 32 || ec + min(k, nd) > a.ecap) { ovf = true; break; }
                    DrawKey dk{a.key, inst, static_cast<uint32_t>(d), v, a.mode, 0};
                    FusedEmit emit{a.s_src, a.s_dst, a.s_dep, e_base + ec, v, static_cast<uint8_t>(d + 1)};
                    uint32_t c;
                    if constexpr (kMode == 2) {
                        CachedDegreePool P{a.col, a.cps, static_cast<uint64_t>(b0), nd, __ldg(a.npos + v), 0, a.bt,
                                           a.wx.head ? 0 : __ldg(a.bt_off + v)};
                        P.wx = a.wx;
                        P.vid = v;
                        const Ctps C = build_ctps(P, tab);
                        c = select_wor(P, C, tab, bm, k, dk, a.a_max, nullptr, emit);
                        probes += P.probes;
                    } else if constexpr (kMode == 1) {
                        DegreePool P{a.col, a.deg, static_cast<uint64_t>(b0), nd, a.ccache};
                        const Ctps C = build_ctps(P, tab);
                        c = select_wor(P, C, tab, bm, k, dk, a.a_max, nullptr, emit);
                        scanned += (a.ccache && C.m) ? 32u * C.m : nd;
                    } else if constexpr (kMode == 6) {
                        VPool<float> P;
                        P.init(a.w, a.col, static_cast<uint64_t>(b0), nd);
                        double* ftab = reinterpret_cast<double*>(tab);
                        const VCtps<float> C = vscan_build<float, 1>(P, ftab, nullptr, 0, [] {});
                        c = vscan_select_wor(P, C, ftab, k, dk, a.a_max, nullptr, emit);
                        scanned += nd;
                    } else {
                        UniformPool P{a.col, static_cast<uint64_t>(b0), nd};
                        const Ctps C = build_ctps(P, tab);
                        c = select_wor(P, C, tab, bm, k, dk, a.a_max, nullptr, emit);
                    }
                    ec += c;
                    ++pools;
            draws += dk.draws;
                }
                if (ovf) break;
            }
            __syncwarp();
            if (d + 1 == a.depth) break;
            // UPDATE (R9): unvisited picks of this level -> next frontier
            for (uint32_t e0 = ec0; e0 < ec; e0 += 32) {
                const uint32_t e = e0 + lane;
                uint32_t u = e < ec ? a.s_dst[e_base + e] : NONE;
                if (u != NONE)
                    for (uint32_t q = 0; q < nv; ++q)
                        if (VIS[q] == u) { u = NONE; break; }
                const unsigned bal = __ballot_sync(FULL, u != NONE);
                const uint32_t pos = nnx + __popc(bal & lanemask_lt());
                if (u != NONE && pos < kF) NX[pos] = u;
                nnx += __popc(bal);
            }
            __syncwarp();
            if (nnx > kF) { ovf = true; break; }
            // sort + unique (set semantics, R10)
            uint32_t P2 = 32;
            while (P2 < nnx) P2 <<= 1;
            for (uint32_t j = nnx + lane; j < P2; j += 32) NX[j] = NONE;
            __syncwarp();
            for (uint32_t kk = 2; kk <= P2; kk <<= 1) {
                for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
                    for (uint32_t idx = lane; idx < P2; idx += 32) {
                        const uint32_t pr = idx ^ jj;
                        if (pr > idx) {
                            const uint32_t x0 = NX[idx], x1 = NX[pr];
                            if ((x0 > x1) == ((idx & kk) == 0)) { NX[idx] = x1; NX[pr] = x0; }
                        }
                    }
                    __syncwarp();
                }
            }
            uint32_t w = 0;
            for (uint32_t j0 = 0; j0 < nnx; j0 += 32) {
                const uint32_t j = j0 + lane;
                const uint32_t u = j < nnx ? NX[j] : NONE;
                const bool keep = u != NONE && (j == 0 || NX[j - 1] != u);
                const unsigned bal = __ballot_sync(FULL, keep);
                if (keep) F[w + __popc(bal & lanemask_lt())] = u;
                w += __popc(bal);
            }
            __syncwarp();
            nf = w;
            if (nv + nf > kVIS) { ovf = true; break; }
            for (uint32_t j = lane; j < nf; j += 32) VIS[nv + j] = F[j];
            nv += nf;
            __syncwarp();
        }
        if (lane == 0) {
            a.cnt[i] = ec;
            if (ovf) atomicOr(a.overflow, 1u);
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (scanned) atomicAdd(a.counters + 0, scanned);
        if (pools) atomicAdd(a.counters + 1, pools);
        if (probes) atomicAdd(a.counters + 2, probes);
        if (draws) atomicAdd(a.counters + 3, draws);
    }
    fused_epilogue<FUSED_WARPS * 32>(a);
}

// Compacts the staging rows into the caller's arrays.  Guarded on the device so the
// host need not wait between the fused kernel and the copy: nothing is written if
// the fused pass overflowed or the output does not fit `capacity`.
__global__ void k_fused_copy(const uint32_t* __restrict__ s_src, const uint32_t* __restrict__ s_dst,
                             const uint8_t* __restrict__ s_dep, uint32_t ecap, const uint64_t* __restrict__ offs,
                             uint64_t n, uint32_t* __restrict__ src, uint32_t* __restrict__ dst, uint8_t* __restrict__ dep,
                             const unsigned* __restrict__ overflow, uint64_t capacity) {
    if (*overflow != 0 || offs[n] > capacity) return;
    const int lane = lane_id();
    for (uint64_t i = global_warp_id(); i < n; i += total_warps()) {
        const uint64_t o = offs[i], c = offs[i + 1] - o;
        for (uint64_t j = lane; j < c; j += 32) {
            src[o + j] = s_src[i * ecap + j];
            dst[o + j] = s_dst[i * ecap + j];
            dep[o + j] = s_dep[i * ecap + j];
        }
    }
}

// ---------------------------------------------------------------- host driver
static int grid_for(const csaw_graph* g, uint64_t n, int per_block = 256) {
    const uint64_t b = (n + per_block - 1) / per_block;
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(b, static_cast<uint64_t>(g->num_sms) * 16)));
}

static int sel_grid(const csaw_graph* g, uint64_t nwork) {
    const uint64_t warps = std::min<uint64_t>(std::max<uint64_t>(nwork, 1), static_cast<uint64_t>(g->num_sms) * 64);
    return static_cast<int>((warps + SEL_WARPS - 1) / SEL_WARPS);
}

template <class T>
static csaw_status lvl_buf(const csaw_graph* g, int l, int k, uint64_t count, T** out) {
    void* p;
    CSAW_TRY(g->scratch.get(SL_LEVEL_BASE + l * 16 + k, sizeof(T) * std::max<uint64_t>(count, 1), &p));
    *out = static_cast<T*>(p);
    return CSAW_OK;
}

// One level of batched sampling in OOM mode (see k_part_count above).
static csaw_status oom_select_level(const csaw_graph* g, const csaw_bias& b, const uint32_t* qv, const uint32_t* qi,
                                    uint64_t nq, const uint32_t* kq, const uint32_t* ub, const uint64_t* eoff,
                                    uint32_t* s_inst, uint32_t* s_src, uint32_t* s_dst, uint32_t d, uint32_t base,
                                    uint2 key, uint32_t a_max, PickRec* glist, uint32_t kmax,
                                    unsigned long long* counters, bool degree_bias, cudaStream_t st) {
    auto& os = const_cast<csaw_graph*>(g)->oomst;
    const uint32_t P = static_cast<uint32_t>(os.P);
    OwnerP own{static_cast<uint64_t>(g->V) / P, static_cast<uint64_t>(g->V) % P};
    void *pc, *pi;
    CSAW_TRY(g->scratch.get(SL_LEVEL_BASE + 253 * 16 + 0, sizeof(uint32_t) * 2 * (P + 1), &pc));
    CSAW_TRY(g->scratch.get(SL_LEVEL_BASE + 253 * 16 + 1, sizeof(uint32_t) * std::max<uint64_t>(nq, 1), &pi));
    uint32_t* cnt = static_cast<uint32_t*>(pc);
    uint32_t* fill = cnt + (P + 1);
    uint32_t* idx = static_cast<uint32_t*>(pi);
    std::vector<uint32_t> hc(2 * (P + 1));   // P is unbounded: pageable staging, synchronised below
    CSAW_CUDA(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * P, st));
    k_part_count<<<grid_for(g, nq), 256, 0, st>>>(qv, nq, own, cnt);
    note_launch();
    CSAW_CUDA(cudaMemcpyAsync(hc.data(), cnt, sizeof(uint32_t) * P, cudaMemcpyDeviceToHost, st));
    CSAW_CUDA(cudaStreamSynchronize(st));
    std::vector<uint64_t> c(P), off(P + 1, 0);
    for (uint32_t p = 0; p < P; ++p) { c[p] = hc[p]; off[p + 1] = off[p] + c[p]; }
    for (uint32_t p = 0; p < P; ++p) hc[P + 1 + p] = static_cast<uint32_t>(off[p]);
    CSAW_CUDA(cudaMemcpyAsync(fill, hc.data() + P + 1, sizeof(uint32_t) * P, cudaMemcpyHostToDevice, st));
    k_part_scatter<<<grid_for(g, nq), 256, 0, st>>>(qv, nq, own, fill, idx);
    note_launch();
    CSAW_CUDA(cudaGetLastError());
    // waves over the partitions with entries (oom_plan_wave: workload-aware, or the
    // round-robin ablation); each partition of the level is sampled exactly once
    std::vector<uint64_t> left(c);
    std::vector<cudaEvent_t> tev;
    cudaEvent_t evs;
    CSAW_CUDA(cudaEventCreateWithFlags(&evs, cudaEventDisableTiming));
    const int blocks_total = g->num_sms * 8;
    for (;;) {
        bool any = false;
        for (uint32_t p = 0; p < P; ++p) any |= left[p] > 0;
        if (!any) break;
        const std::vector<WavePick> wave = oom_plan_wave(os, left);
        CSAW_CUDA(cudaEventRecord(evs, st));
        for (const WavePick& w : wave)
            if (w.fresh) CSAW_TRY(oom_load(g, w.p, w.slot, evs, tev));
        uint64_t wave_total = 0;
        for (const WavePick& w : wave) wave_total += left[w.p];
        for (const WavePick& w : wave) {
            const int32_t p = w.p;
            cudaStream_t ss = os.streams[w.slot % os.S];
            CSAW_CUDA(cudaStreamWaitEvent(ss, evs, 0));
            const int blocks = oom_blocks(os, blocks_total, left[p], wave_total, wave.size(), SEL_WARPS);
            const uint32_t* colp = os.d_slots + static_cast<int64_t>(w.slot) * os.slot_edges - os.ebeg[p];
            SelArgs sa{g->row_ptr, colp, g->deg, qv, qi, nq, kq, ub, eoff, s_inst, s_src, s_dst, d, base, key, a_max,
                       glist, kmax, counters, nullptr, nullptr, nullptr, nullptr, static_cast<uint32_t>(b.migration),
                       idx + off[p], c[p], g->ccache, WixPtrs{}};
            CSAW_TRY(hot_begin(g, ss));
            if (degree_bias) k_ns_select<1><<<blocks, SEL_WARPS * 32, 0, ss>>>(sa);
            else k_ns_select<0><<<blocks, SEL_WARPS * 32, 0, ss>>>(sa);
            note_launch();
            CSAW_CUDA(cudaGetLastError());
            CSAW_TRY(hot_end(g, ss));
            left[p] = 0;
        }
        for (int s = 0; s < os.S; ++s) {
            CSAW_CUDA(cudaEventRecord(evs, os.streams[s]));
            CSAW_CUDA(cudaStreamWaitEvent(st, evs, 0));
        }
    }
    oom_account_transfers(g, tev);
    cudaEventDestroy(evs);
    return CSAW_OK;
}

// Fused path: returns CSAW_OK when done, CSAW_ERR_CAPACITY / OUT_OF_RANGE as usual, and
// FUSED_FALLBACK when the batched level-synchronous driver must run instead.
constexpr csaw_status FUSED_FALLBACK = static_cast<csaw_status>(-1);

// vertex heads usable by the cached sampling pools (leaf fanout 128 only)
static WixPtrs wix_ptrs(const csaw_graph* g) {
    WixPtrs w;
    if (g->whead && g->wix_leaf == 128 && !(g->flags & CSAW_GRAPH_SAMPLE_NO_HEADS)) {
        w.head = g->whead; w.c32 = g->c32; w.col = g->wcol; w.inn = g->winn;
    }
    return w;
}

static csaw_status run_sample_fused(const csaw_graph* g, const csaw_bias& b, const int32_t* fanout, int32_t depth,
                                    const uint32_t* d_seeds, uint64_t n, uint64_t base, uint64_t seed,
                                    uint64_t* d_offsets, uint32_t* src, uint32_t* dst, uint8_t* dep, int64_t capacity,
                                    int64_t* num_edges, bool out_on_device, cudaStream_t st,
                                    uint64_t* offs_host = nullptr) {
    const bool layer = b.kind == CSAW_BIAS_LAYER;
    const bool ff = b.kind == CSAW_BIAS_FOREST_FIRE;
    // per-instance staging capacity from the fanouts (forest fire: a fixed budget)
    double ecap_d = 0;
    if (ff) {
        ecap_d = 512;
    } else {
        double level = 1;
        for (int d = 0; d < depth; ++d) {
            if (fanout[d] > 32) return FUSED_FALLBACK;
            level = layer ? fanout[d] : level * fanout[d];
            ecap_d += level;
        }
    }
    if (ecap_d > 2048 || n == 0 || depth > 16) return FUSED_FALLBACK;
    const uint32_t ecap = std::max<uint32_t>(1, static_cast<uint32_t>(ecap_d));
    void *pc, *ps, *pd, *pe, *pk;
    CSAW_TRY(g->scratch.get(SL_COUNTS, 256, &pc));
    unsigned long long* counters = static_cast<unsigned long long*>(pc);
    unsigned* ovf = reinterpret_cast<unsigned*>(counters + 12);
    CSAW_TRY(g->scratch.get(SL_SRC + 200, sizeof(uint32_t) * n * ecap, &ps));
    CSAW_TRY(g->scratch.get(SL_SRC + 201, sizeof(uint32_t) * n * ecap, &pd));
    CSAW_TRY(g->scratch.get(SL_SRC + 202, static_cast<size_t>(n) * ecap, &pe));
    CSAW_TRY(g->scratch.get(SL_SRC + 203, sizeof(uint64_t) * n, &pk));
    void* hmb;
    CSAW_TRY(g->pinned.get(4096, &hmb));
    volatile uint64_t* hbox = static_cast<volatile uint64_t*>(hmb);
    CSAW_CUDA(cudaMemsetAsync(counters, 0, 256, st));
    CSAW_TRY(stats_begin(g, st));
    FusedArgs a;
    a.rp = g->row_ptr; a.col = g->oom ? g->oomst.src_col : g->col; a.deg = g->deg; a.cps = g->cps; a.npos = g->npos; a.bt = g->bt;
    a.bt_off = g->bt_off; a.seeds = d_seeds; a.n = n; a.depth = depth;
    for (int d = 0; d < 16; ++d) a.fanout[d] = (d < depth && !ff) ? fanout[d] : 0;
    a.theta = ff ? static_cast<uint64_t>(std::floor(b.pf * 4294967296.0)) : 0;
    a.base = static_cast<uint32_t>(base);
    a.key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    a.a_max = b.a_max ? static_cast<uint32_t>(b.a_max) : 64u;
    a.ecap = ecap;
    a.s_src = static_cast<uint32_t*>(ps); a.s_dst = static_cast<uint32_t*>(pd); a.s_dep = static_cast<uint8_t*>(pe);
    a.cnt = static_cast<uint64_t*>(pk);
    a.overflow = ovf;
    a.counters = counters;
    a.offs = d_offsets;
    a.offs_host = offs_host;
    a.ccache = g->ccache;
    a.wx = wix_ptrs(g);
    a.w = g->w;
    a.done = reinterpret_cast<unsigned*>(counters + 13);   // zeroed by the memset above
    a.report = const_cast<uint64_t*>(hbox);
    a.V = g->V;
    a.mode = static_cast<uint32_t>(b.migration);
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + FUSED_WARPS - 1) / FUSED_WARPS,
                                                                                static_cast<uint64_t>(g->num_sms) * 16)));
    CSAW_TRY(hot_begin(g, st));
    if (layer) {
        if (g->cps) k_sample_fused<5><<<grid, FUSED_WARPS * 32, 0, st>>>(a);
        else k_sample_fused<4><<<grid, FUSED_WARPS * 32, 0, st>>>(a);
    } else if (ff) {
        k_sample_fused<3><<<grid, FUSED_WARPS * 32, 0, st>>>(a);
    } else if (b.kind == CSAW_BIAS_DEGREE) {
        if (g->cps) k_sample_fused<2><<<grid, FUSED_WARPS * 32, 0, st>>>(a);
        else k_sample_fused<1><<<grid, FUSED_WARPS * 32, 0, st>>>(a);
    } else if (b.kind == CSAW_BIAS_WEIGHT) {
        k_sample_fused<6><<<grid, FUSED_WARPS * 32, 0, st>>>(a);
    } else {
        k_sample_fused<0><<<grid, FUSED_WARPS * 32, 0, st>>>(a);
    }
    note_launch();
    CSAW_CUDA(cudaGetLastError());
    CSAW_TRY(hot_end(g, st));
    if (out_on_device && capacity > 0) {   // no host round trip before the copy
        k_fused_copy<<<grid, FUSED_WARPS * 32, 0, st>>>(a.s_src, a.s_dst, a.s_dep, ecap, d_offsets, n, src, dst, dep, ovf,
                                                         static_cast<uint64_t>(capacity));
        note_launch();
        CSAW_CUDA(cudaGetLastError());
    }
    CSAW_TRY(stats_end(g, st));
    CSAW_CUDA(cudaStreamSynchronize(st));   // the fused kernel's last block wrote the report
    const unsigned flags = static_cast<unsigned>(hbox[0] & 0xFFFFFFFFu);
    if (flags & 2u) return fail(CSAW_ERR_OUT_OF_RANGE, "a seed vertex is >= num_vertices");
    if (flags & 1u) return FUSED_FALLBACK;
    const uint64_t nedges = hbox[1];
    *num_edges = static_cast<int64_t>(nedges);
    g->stats.sampled_edges = nedges;
    g->stats.neighbours_scanned = hbox[2];
    g->stats.pools = hbox[3];
    g->stats.cache_probes = hbox[4];
    g->stats.draws = hbox[5];
    if (static_cast<int64_t>(nedges) > capacity)
        return fail(CSAW_ERR_CAPACITY, "output capacity " + std::to_string(capacity) + " < required " +
                                           std::to_string(nedges));
    if (!out_on_device && nedges > 0) {   // host output: compact into scratch, then copy down
        void *p0, *p1, *p2;
        CSAW_TRY(g->scratch.get(SL_SRC, sizeof(uint32_t) * nedges, &p0));
        CSAW_TRY(g->scratch.get(SL_DST, sizeof(uint32_t) * nedges, &p1));
        CSAW_TRY(g->scratch.get(SL_DEP, nedges, &p2));
        uint32_t* osrc = static_cast<uint32_t*>(p0);
        uint32_t* odst = static_cast<uint32_t*>(p1);
        uint8_t* odep = static_cast<uint8_t*>(p2);
        k_fused_copy<<<grid, FUSED_WARPS * 32, 0, st>>>(a.s_src, a.s_dst, a.s_dep, ecap, d_offsets, n, osrc, odst, odep,
                                                         ovf, static_cast<uint64_t>(nedges));
        note_launch();
        CSAW_CUDA(cudaGetLastError());
        CSAW_CUDA(cudaMemcpyAsync(src, osrc, sizeof(uint32_t) * nedges, cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaMemcpyAsync(dst, odst, sizeof(uint32_t) * nedges, cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaMemcpyAsync(dep, odep, nedges, cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaStreamSynchronize(st));
    }
    return CSAW_OK;
}

csaw_status run_sample(const csaw_graph* g, const csaw_bias& b, const int32_t* fanout, int32_t depth,
                       const uint32_t* d_seeds, int64_t n_i64, uint64_t base, uint64_t seed, uint64_t* d_offsets,
                       uint32_t* src, uint32_t* dst, uint8_t* dep, int64_t capacity, int64_t* num_edges,
                       bool out_on_device, cudaStream_t st, PinnedOut* pinned) {
    if (!g->force_batched && (!g->oom || g->oomst.zerocopy) && b.kind != CSAW_BIAS_SNOWBALL) {
        // pinned host outputs: the fused copy writes each instance's contiguous segment over the
        // host link (coalesced), so no staging and no copy after the kernels
        const bool direct = !out_on_device && pinned != nullptr && pinned->src && pinned->dst && pinned->dep;
        uint64_t* offs_host = pinned ? pinned->offs : nullptr;
        const csaw_status s = run_sample_fused(g, b, fanout, depth, d_seeds, static_cast<uint64_t>(n_i64), base, seed,
                                               d_offsets, direct ? pinned->src : src, direct ? pinned->dst : dst,
                                               direct ? pinned->dep : dep, capacity, num_edges,
                                               out_on_device || direct, st, offs_host);
        if (s != FUSED_FALLBACK) {
            if (offs_host) pinned->offs_done = true;
            return s;
        }
    }
    return run_sample_levels(g, b, fanout, depth, d_seeds, n_i64, base, seed, d_offsets, src, dst, dep, capacity,
                             num_edges, out_on_device, st);
}

// Level-synchronous batched driver (general path).
csaw_status run_sample_levels(const csaw_graph* g, const csaw_bias& b, const int32_t* fanout, int32_t depth,
                       const uint32_t* d_seeds, int64_t n_i64, uint64_t base, uint64_t seed, uint64_t* d_offsets,
                       uint32_t* src, uint32_t* dst, uint8_t* dep, int64_t capacity, int64_t* num_edges,
                       bool out_on_device, cudaStream_t st) {
    const uint64_t n = static_cast<uint64_t>(n_i64);
    const bool layer = b.kind == CSAW_BIAS_LAYER;
    const bool ff = b.kind == CSAW_BIAS_FOREST_FIRE;
    const bool snow = b.kind == CSAW_BIAS_SNOWBALL;   // uniform bias, k = all (select-all path, R8)
    const bool degree_bias = b.kind == CSAW_BIAS_DEGREE;
    // zero-copy OOM mode reads col_idx in place from pinned host memory (UVA)
    const uint32_t* colz = g->oom ? g->oomst.src_col : g->col;
    const uint32_t a_max = b.a_max ? static_cast<uint32_t>(b.a_max) : 64u;
    const uint2 key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    const uint64_t theta = ff ? static_cast<uint64_t>(std::floor(b.pf * 4294967296.0)) : 0;
    const int vbits = std::max(1, bits_for(static_cast<uint64_t>(std::max<int64_t>(g->V, 1) - 1)));
    const int ibits = std::max(1, bits_for(n > 0 ? n - 1 : 0));
    if (vbits + ibits + 1 > 64) return fail(CSAW_ERR_UNSUPPORTED, "instance/vertex key does not fit 64 bits");
    const int nbits = vbits + ibits + 1;

    // small pinned host mailbox for per-level counts
    void* hmb;
    CSAW_TRY(g->pinned.get(4096, &hmb));
    volatile uint64_t* hbox = static_cast<volatile uint64_t*>(hmb);

    void *cnt_v, *part_v, *err_v;
    CSAW_TRY(g->scratch.get(SL_COUNTS, 256, &cnt_v));
    unsigned long long* counters = static_cast<unsigned long long*>(cnt_v);
    unsigned* err = reinterpret_cast<unsigned*>(counters + 8);
    unsigned* kmaxd = reinterpret_cast<unsigned*>(counters + 9);
    uint64_t* nq_next = reinterpret_cast<uint64_t*>(counters + 10);
    CSAW_TRY(g->scratch.get(SL_TMP2, sizeof(uint64_t) * (SCAN_MAX_GRID + 8), &part_v));
    uint64_t* part = static_cast<uint64_t*>(part_v);
    (void)err_v;
    CSAW_CUDA(cudaMemsetAsync(counters, 0, 256, st));
    CSAW_TRY(stats_begin(g, st));

    std::vector<LevelDesc> hlev(depth + 1);
    std::vector<uint64_t> totals(depth, 0);
    std::vector<uint32_t*> sinst(depth), ssrc(depth), sdst(depth);

    // level 0 queue = seeds
    uint32_t *qv, *qi;
    uint64_t* inst_off;
    CSAW_TRY(lvl_buf(g, 0, 0, n, &qv));
    CSAW_TRY(lvl_buf(g, 0, 1, n, &qi));
    CSAW_TRY(lvl_buf(g, 0, 2, n + 1, &inst_off));
    k_init_queue<<<grid_for(g, n + 1), 256, 0, st>>>(d_seeds, n, g->V, qv, qi, inst_off, err);
    note_launch();
    CSAW_CUDA(cudaGetLastError());
    uint64_t nq = n;

    // device copy of level descriptors (for the visited test / counts)
    LevelDesc* dlev;
    CSAW_TRY(lvl_buf(g, 255, 15, depth + 1, &dlev));

    for (int l = 0; l < depth; ++l) {
        hlev[l].qv = qv;
        hlev[l].inst_off = inst_off;
        hlev[l].layer = layer ? 1 : 0;
        const uint64_t nwork = layer ? n : nq;
        uint32_t *ub, *kq = nullptr;
        uint64_t* eoff;
        CSAW_TRY(lvl_buf(g, l, 3, nwork, &ub));
        CSAW_TRY(lvl_buf(g, l, 4, nwork + 1, &eoff));
        uint64_t* qpref = nullptr;
        const uint32_t fan = ff ? 0u : snow ? 0xFFFFFFFFu : static_cast<uint32_t>(fanout[l]);
        CSAW_CUDA(cudaMemsetAsync(kmaxd, 0, sizeof(unsigned), st));
        if (layer) {
            CSAW_TRY(lvl_buf(g, l, 5, nq + 1, &qpref));
            CSAW_TRY(device_scan(DegOfQueue{g->row_ptr, qv}, nq, ScanToArray{qpref}, part, st));
            k_layer_bound<<<grid_for(g, n), 256, 0, st>>>(inst_off, qpref, n, fan, ub, err, kmaxd);
            note_launch();
        } else {
            CSAW_TRY(lvl_buf(g, l, 5, nq, &kq));
            if (nq > 0) {
                note_launch();
                k_ns_bound<<<grid_for(g, nq), 256, 0, st>>>(g->row_ptr, qv, qi, nq, ff ? 1 : 0, fan, theta,
                                                            static_cast<uint32_t>(l), static_cast<uint32_t>(base), key,
                                                            ub, kq, kmaxd);
            }
        }
        CSAW_CUDA(cudaGetLastError());
        CSAW_TRY(device_scan(U32Val{ub}, nwork, ScanToArray{eoff}, part, st));
        unsigned* segmaxd = kmaxd + 1;
        CSAW_CUDA(cudaMemsetAsync(segmaxd, 0, sizeof(unsigned), st));
        if (l + 1 < depth && n > 0) {
            k_segmax<<<grid_for(g, n), 256, 0, st>>>(eoff, inst_off, layer ? 1 : 0, n, segmaxd);
            note_launch();
        }
        // read total staged entries + kmax + error flags + largest per-instance segment
        hbox[1] = 0; hbox[2] = 0; hbox[8] = 0;
        CSAW_CUDA(cudaMemcpyAsync((void*)&hbox[8], segmaxd, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaMemcpyAsync((void*)&hbox[0], eoff + nwork, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaMemcpyAsync((void*)&hbox[1], kmaxd, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaMemcpyAsync((void*)&hbox[2], err, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaStreamSynchronize(st));
        const uint64_t total = hbox[0];
        const uint32_t kmax = static_cast<uint32_t>(hbox[1] & 0xFFFFFFFFu);
        const unsigned errs = static_cast<unsigned>(hbox[2] & 0xFFFFFFFFu);
        const uint32_t segmax = static_cast<uint32_t>(hbox[8] & 0xFFFFFFFFu);
        if (errs & ERR_SEED_RANGE) return fail(CSAW_ERR_OUT_OF_RANGE, "a seed vertex is >= num_vertices");
        if (errs & ERR_POOL_TOO_BIG) return fail(CSAW_ERR_UNSUPPORTED, "a layer pool has >= 2^32-64 candidates");
        if (kmax >= (1u << 14)) return fail(CSAW_ERR_UNSUPPORTED, "a pool needs >= 2^14 picks (draw counter field)");
        totals[l] = total;
        uint32_t *s_inst, *s_src, *s_dst;
        CSAW_TRY(lvl_buf(g, l, 6, total, &s_inst));
        CSAW_TRY(lvl_buf(g, l, 7, total, &s_src));
        CSAW_TRY(lvl_buf(g, l, 8, total, &s_dst));
        sinst[l] = s_inst; ssrc[l] = s_src; sdst[l] = s_dst;
        PickRec* glist = nullptr;
        const int sgrid = sel_grid(g, nwork);
        if (kmax > 32) {
            void* p;
            CSAW_TRY(g->scratch.get(SL_GLIST, sizeof(PickRec) * kmax * static_cast<uint64_t>(sgrid) * SEL_WARPS, &p));
            glist = static_cast<PickRec*>(p);
        }
        if (nwork > 0 && total > 0 && g->oom && !g->oomst.zerocopy) {
            CSAW_TRY(oom_select_level(g, b, qv, qi, nq, kq, ub, eoff, s_inst, s_src, s_dst, static_cast<uint32_t>(l),
                                      static_cast<uint32_t>(base), key, a_max, glist, kmax, counters, degree_bias, st));
        } else if (nwork > 0 && total > 0) {
            CSAW_TRY(hot_begin(g, st));
            note_launch();
            if (layer) {
                LayerArgs la{g->row_ptr, colz, g->deg, qv, inst_off, qpref, n, fan, ub, eoff, s_inst, s_src, s_dst,
                             static_cast<uint32_t>(l), static_cast<uint32_t>(base), key, a_max, glist, kmax, counters,
                             g->cps, g->npos, g->bt, g->bt_off, static_cast<uint32_t>(b.migration), wix_ptrs(g)};
                if (g->cps) k_layer_select<true><<<sgrid, SEL_WARPS * 32, 0, st>>>(la);
                else k_layer_select<false><<<sgrid, SEL_WARPS * 32, 0, st>>>(la);
            } else {
                SelArgs sa{g->row_ptr, colz, g->deg, qv, qi, nq, kq, ub, eoff, s_inst, s_src, s_dst,
                           static_cast<uint32_t>(l), static_cast<uint32_t>(base), key, a_max, glist, kmax, counters,
                           g->cps, g->npos, g->bt, g->bt_off, static_cast<uint32_t>(b.migration), nullptr, 0,
                           g->ccache, wix_ptrs(g)};
                sa.w = g->w;
                if (b.kind == CSAW_BIAS_WEIGHT) k_ns_select<3><<<sgrid, SEL_WARPS * 32, 0, st>>>(sa);
                else if (degree_bias && g->cps) k_ns_select<2><<<sgrid, SEL_WARPS * 32, 0, st>>>(sa);
                else if (degree_bias) k_ns_select<1><<<sgrid, SEL_WARPS * 32, 0, st>>>(sa);
                else k_ns_select<0><<<sgrid, SEL_WARPS * 32, 0, st>>>(sa);
            }
            CSAW_CUDA(cudaGetLastError());
            CSAW_TRY(hot_end(g, st));
        }
        // rank of valid staged entries (final assembly)
        uint64_t* rank;
        CSAW_TRY(lvl_buf(g, l, 9, total + 1, &rank));
        CSAW_TRY(device_scan(ValidVal{s_dst}, total, ScanToArray{rank}, part, st));
        hlev[l].eoff = eoff;
        hlev[l].rank = rank;
        uint64_t* lvlbase;
        CSAW_TRY(lvl_buf(g, l, 10, n, &lvlbase));
        hlev[l].lvlbase = lvlbase;

        if (l + 1 == depth) break;
        // ---- UPDATE: next frontier (visited post-filter, set semantics)
        CSAW_CUDA(cudaMemcpyAsync(dlev, hlev.data(), sizeof(LevelDesc) * (l + 1), cudaMemcpyHostToDevice, st));
        if (segmax <= FSEG) {
            // segmented path: per-instance shared-memory sort / dedup (no global sort)
            VisitedArgs va{d_seeds, dlev, l};
            uint32_t *tmpq, *nqv, *nqi;
            uint64_t *cntv, *noff;
            CSAW_TRY(lvl_buf(g, l, 11, total, &tmpq));
            CSAW_TRY(lvl_buf(g, l, 12, n, &cntv));
            CSAW_TRY(lvl_buf(g, l + 1, 2, n + 1, &noff));
            const int fg = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + FSEG_WARPS - 1) / FSEG_WARPS,
                                                                                      static_cast<uint64_t>(g->num_sms) * 16)));
            if (n > 0) {
                k_frontier_seg<<<fg, FSEG_WARPS * 32, 0, st>>>(eoff, inst_off, layer ? 1 : 0, s_dst, va, n, tmpq, cntv);
                note_launch();
            }
            CSAW_TRY(device_scan(U64Val{cntv}, n, ScanToArray{noff}, part, st));
            CSAW_CUDA(cudaMemcpyAsync((void*)&hbox[3], noff + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
            CSAW_CUDA(cudaStreamSynchronize(st));
            nq = hbox[3];
            CSAW_TRY(lvl_buf(g, l + 1, 0, nq, &nqv));
            CSAW_TRY(lvl_buf(g, l + 1, 1, nq, &nqi));
            if (n > 0 && nq > 0) {
                k_frontier_compact<<<fg, FSEG_WARPS * 32, 0, st>>>(eoff, inst_off, layer ? 1 : 0, tmpq, noff, n, nqv, nqi);
                note_launch();
            }
            CSAW_CUDA(cudaGetLastError());
            qv = nqv; qi = nqi; inst_off = noff;
            continue;
        }
        // general path (an instance staged > FSEG picks): global LSD radix sort of (instance, vertex)
        uint64_t *keys, *alt, *hist, *hoffs;
        CSAW_TRY(lvl_buf(g, l, 11, total, &keys));
        CSAW_TRY(lvl_buf(g, l, 12, total, &alt));
        const int rg = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(512, (total + 4095) / 4096)));
        CSAW_TRY(lvl_buf(g, l, 13, static_cast<uint64_t>(256) * rg, &hist));
        CSAW_TRY(lvl_buf(g, l, 14, static_cast<uint64_t>(256) * rg + 1, &hoffs));
        VisitedArgs va{d_seeds, dlev, l};
        if (total > 0) { k_cand<<<grid_for(g, total), 256, 0, st>>>(s_inst, s_dst, total, va, vbits, keys); note_launch(); }
        CSAW_CUDA(cudaGetLastError());
        uint64_t* sorted = keys;
        CSAW_TRY(radix_sort_u64(keys, alt, total, nbits, hist, hoffs, part, &sorted, st));
        uint32_t *nqv, *nqi;
        uint64_t* noff;
        CSAW_TRY(lvl_buf(g, l + 1, 0, total, &nqv));
        CSAW_TRY(lvl_buf(g, l + 1, 1, total, &nqi));
        CSAW_TRY(lvl_buf(g, l + 1, 2, n + 1, &noff));
        CSAW_TRY(device_scan(UniqueFlag{sorted}, total, CompactQueue{sorted, nqv, nqi, nq_next, vbits}, part, st));
        CSAW_CUDA(cudaMemcpyAsync((void*)&hbox[3], nq_next, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaStreamSynchronize(st));
        nq = hbox[3];
        k_inst_off<<<grid_for(g, n + 1), 256, 0, st>>>(nqi, nq, n, noff);
        note_launch();
        CSAW_CUDA(cudaGetLastError());
        qv = nqv; qi = nqi; inst_off = noff;
    }

    // ---- final assembly: per-instance offsets in canonical (depth, src, dst) order
    CSAW_CUDA(cudaMemcpyAsync(dlev, hlev.data(), sizeof(LevelDesc) * depth, cudaMemcpyHostToDevice, st));
    uint64_t* tot;
    CSAW_TRY(lvl_buf(g, 254, 0, n, &tot));
    if (n > 0) { k_counts<<<grid_for(g, n), 256, 0, st>>>(dlev, depth, n, tot); note_launch(); }
    CSAW_TRY(device_scan(U64Val{tot}, n, ScanToArray{d_offsets}, part, st));
    CSAW_CUDA(cudaMemcpyAsync((void*)&hbox[4], d_offsets + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    CSAW_CUDA(cudaMemcpyAsync((void*)&hbox[5], counters, sizeof(uint64_t) * 4, cudaMemcpyDeviceToHost, st));
    CSAW_CUDA(cudaStreamSynchronize(st));
    const uint64_t nedges = hbox[4];
    *num_edges = static_cast<int64_t>(nedges);
    g->stats.sampled_edges = nedges;
    g->stats.neighbours_scanned = hbox[5];
    g->stats.pools = hbox[6];
    g->stats.cache_probes = hbox[7];
    g->stats.draws = hbox[8];
    if (static_cast<int64_t>(nedges) > capacity) {
        CSAW_TRY(stats_end(g, st));
        return fail(CSAW_ERR_CAPACITY, "output capacity " + std::to_string(capacity) + " < required " +
                                           std::to_string(nedges));
    }
    uint32_t *osrc = src, *odst = dst;
    uint8_t* odep = dep;
    if (!out_on_device && nedges > 0) {
        void *p0, *p1, *p2;
        CSAW_TRY(g->scratch.get(SL_SRC, sizeof(uint32_t) * nedges, &p0));
        CSAW_TRY(g->scratch.get(SL_DST, sizeof(uint32_t) * nedges, &p1));
        CSAW_TRY(g->scratch.get(SL_DEP, nedges, &p2));
        osrc = static_cast<uint32_t*>(p0); odst = static_cast<uint32_t*>(p1); odep = static_cast<uint8_t*>(p2);
    }
    for (int l = 0; l < depth; ++l) {
        if (totals[l] == 0) continue;
        k_write<<<grid_for(g, totals[l]), 256, 0, st>>>(hlev[l], l + 1, sinst[l], ssrc[l], sdst[l], totals[l],
                                                         d_offsets, osrc, odst, odep);
        note_launch();
    }
    CSAW_CUDA(cudaGetLastError());
    CSAW_TRY(stats_end(g, st));
    if (!out_on_device && nedges > 0) {
        CSAW_CUDA(cudaMemcpyAsync(src, osrc, sizeof(uint32_t) * nedges, cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaMemcpyAsync(dst, odst, sizeof(uint32_t) * nedges, cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaMemcpyAsync(dep, odep, nedges, cudaMemcpyDeviceToHost, st));
    }
    CSAW_CUDA(cudaStreamSynchronize(st));
    return CSAW_OK;
}

}  // namespace csaw
