// select.cuh — warp-centric biased selection (the paper's Select, §4.1-4.2).
//
// One warp owns one candidate pool (inter-warp parallelism).  The
// warp evaluates the pool's biases (EDGEBIAS / VERTEXBIAS, Eq. 2-3), builds an
// exact integer CTPS with a Kogge-Stone __shfl_up_sync scan (Eq. 1, P:477-480;
// F = S/T is never formed, reading R6), draws counter-based Philox randoms and
// inverse-transform-searches the CTPS.  Without replacement, lane j
// owns pick j; collisions are detected with a strided shared-memory
// bitmap plus __match_any_sync, and migrated with bipartite region
// search (box steps 1-5) using a fresh draw over the reduced space
// (reading R1).  Picks are resolved in lane order so the result equals the
// sequential definition (reading R3): the longest prefix of lanes whose
// attempt-0 candidates are free finalises at once; the first colliding lane
// runs BRS serially with the whole warp helping its searches.
//
// CTPS storage (shared memory, per warp): pools of n <= TAB candidates keep the
// full inclusive prefix S[1..n]; larger pools keep one cumulative total per
// chunk of m rows (m a multiple of U, <= TAB chunks) and re-scan a chunk to
// locate a draw inside it -- two-level ITS, bit-identical to a flat search.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "wix.cuh"

namespace csaw {

constexpr int TAB = 256;          // chunk-table entries per warp (2 KB of u64)
constexpr int BM_WORDS = 256;     // strided bitmap words per warp
constexpr uint32_t BM_BITS = BM_WORDS * 32u;
constexpr int U = 8;              // rows (of 32 candidates) in flight per warp
constexpr uint32_t CACHED = 0xFFFFFFFFu;   // Ctps::m marker: the pool searches a cached CTPS

struct Region {
    uint32_t s;      // pool index
    uint32_t b;      // bias b_s
    uint64_t lo;     // S_s (exclusive prefix)
    uint32_t item;   // pool item at s (vertex id), NONE if not fetched
};

struct Ctps {
    uint32_t n;      // pool length
    uint32_t m;      // rows per chunk; 0 = full table (n <= TAB)
    uint32_t nch;    // table entries used
    uint32_t npos;   // candidates with b > 0
    uint64_t T;      // total bias S_n
};

// Taken-pick record kept in per-warp global scratch when k > 32 (several passes).
struct PickRec {
    uint32_t s;
    uint32_t b;
    uint64_t lo;
};

// ---------------------------------------------------------------- CTPS build (pass 1)
// Pool concept (warp-collective unless noted):
//   uint32_t n;
//   static constexpr bool kClosedForm;     // unit biases: S_i = i, no scan
//   void seek(uint32_t row0);              // start a sequential run of rows at row0
//   void load_rows<NR>(row0, key[NR], b[NR]);  // rows row0..row0+NR-1, in increasing order
//   uint32_t item(uint32_t i) const;       // lane-local random access
struct DegreePool;

// Chunk-total cache (capi.cu build_ccache): for a row of d > TAB candidates, the chunk
// prefix sums this scan would produce (same m, same chunks) followed by npos, at
// ccache[row start / 64 ...].  Rows are disjoint there: the gap to the next row,
// floor(d / 64), exceeds nch + 1 <= d / 256 + 3 for d > 256.
__device__ __forceinline__ uint32_t ctps_chunk_rows(uint32_t nrows) {
    uint32_t m = (nrows + TAB - 1) / TAB;
    return ((m + U - 1) / U) * U;
}

template <class Pool>
__device__ __forceinline__ Ctps build_ctps(Pool& P, uint64_t* __restrict__ tab) {
    const int lane = lane_id();
    Ctps c;
    c.n = P.n;
    if constexpr (Pool::kClosedForm) {
        c.m = 0; c.nch = 0; c.npos = P.n; c.T = P.n;
        return c;
    }
    if constexpr (Pool::kCached) {   // static-bias CTPS cache: T and npos are read, not scanned
        c.m = CACHED; c.nch = 0; c.T = P.total(); c.npos = P.npos_count();
        return c;
    }
    const uint32_t n = P.n;
    const uint32_t nrows = (n + 31) >> 5;
    uint64_t carry = 0;
    uint32_t npos = 0;
    P.seek(0);
    if (n <= static_cast<uint32_t>(TAB)) {
        c.m = 0;
        c.nch = n;
        for (uint32_t r0 = 0; r0 < nrows; r0 += U) {
            uint32_t key[U], b[U];
            P.template load_rows<U>(r0, key, b);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (r0 + u < nrows) {
                    const uint64_t incl = warp_incl_scan(b[u]) + carry;
                    const uint32_t i = (r0 + u) * 32 + lane;
                    if (i < n) tab[i] = incl;
                    carry = __shfl_sync(FULL, incl, 31);
                    npos += __popc(__ballot_sync(FULL, b[u] > 0));
                }
            }
        }
    } else {
        const uint32_t m = ctps_chunk_rows(nrows);
        c.m = m;
        c.nch = (nrows + m - 1) / m;
        if constexpr (std::is_same<Pool, DegreePool>::value) {
            if (P.ccache) {   // static degree bias: the chunk table is read, not scanned
                const uint64_t* cc = P.ccache + P.beg / 64;
                for (uint32_t i = lane; i < c.nch; i += 32) tab[i] = __ldg(cc + i);
                c.T = __ldg(cc + c.nch - 1);
                c.npos = static_cast<uint32_t>(__ldg(cc + c.nch));
                __syncwarp();
                return c;
            }
        }
        const uint32_t groups_per_chunk = m / U;
        uint32_t g = 0, chunk = 0;
        uint64_t acc = 0;
        for (uint32_t r0 = 0; r0 < nrows; r0 += U) {
            uint32_t key[U], b[U];
            P.template load_rows<U>(r0, key, b);
            unsigned pos = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc += b[u];
                pos += __popc(__ballot_sync(FULL, b[u] > 0));
            }
            npos += pos;
            if (++g == groups_per_chunk || r0 + U >= nrows) {
                carry += warp_sum(acc);
                if (lane == 0) tab[chunk] = carry;
                ++chunk;
                acc = 0;
                g = 0;
            }
        }
    }
    c.npos = npos;
    c.T = carry;
    __syncwarp();
    return c;
}

// ---------------------------------------------------------------- inverse transform search
// Lane-local search of a full table (n <= TAB): first i with S[i+1] > x.
__device__ __forceinline__ Region its_table(const uint64_t* __restrict__ tab, uint32_t n, uint64_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (tab[mid] > x) hi = mid; else lo = mid + 1;
    }
    Region r;
    r.s = lo;
    r.lo = lo ? tab[lo - 1] : 0;
    r.b = static_cast<uint32_t>(tab[lo] - r.lo);
    r.item = NONE;
    return r;
}

// Warp-collective search for a warp-uniform x (any table layout).
template <class Pool>
__device__ __forceinline__ Region its_uniform(Pool& P, const Ctps& C, const uint64_t* __restrict__ tab, uint64_t x) {
    if constexpr (Pool::kClosedForm) {
        Region r;
        r.s = static_cast<uint32_t>(x); r.lo = x; r.b = 1; r.item = NONE;
        return r;
    } else if constexpr (Pool::kCached) {
        return P.search(x);
    } else {
        if (C.m == 0) return its_table(tab, C.n, x);
        // chunk: first c with tab[c] > x (all lanes search redundantly: broadcast reads)
        uint32_t lo = 0, hi = C.nch;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (tab[mid] > x) hi = mid; else lo = mid + 1;
        }
        const uint32_t c = lo;
        uint64_t base = c ? tab[c - 1] : 0;
        const uint32_t nrows = (C.n + 31) >> 5;
        const uint32_t rbeg = c * C.m;
        const uint32_t rend = min(rbeg + C.m, nrows);
        P.seek(rbeg);
        for (uint32_t r0 = rbeg; r0 < rend; r0 += U) {
            uint32_t key[U], b[U];
            P.template load_rows<U>(r0, key, b);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t incl = warp_incl_scan(b[u]);
                const uint64_t tot = __shfl_sync(FULL, incl, 31);
                if (base + tot > x) {
                    const unsigned hit = __ballot_sync(FULL, base + incl > x);
                    const int f = __ffs(hit) - 1;
                    Region r;
                    r.s = (r0 + u) * 32 + f;
                    r.b = __shfl_sync(FULL, b[u], f);
                    r.lo = base + __shfl_sync(FULL, incl, f) - r.b;
                    r.item = __shfl_sync(FULL, key[u], f);
                    return r;
                }
                base += tot;
            }
        }
        Region r;  // unreachable for x < T
        r.s = NONE; r.b = 0; r.lo = 0; r.item = NONE;
        return r;
    }
}

// ---------------------------------------------------------------- selection with replacement
// One draw (walks): x = below(U, T), s = its(x).  Returns the picked item.
template <class Pool>
__device__ __forceinline__ uint32_t select_wr(Pool& P, const Ctps& C, const uint64_t* __restrict__ tab,
                                              uint64_t U64) {
    if (C.T == 0) return NONE;
    const uint64_t x = below(U64, C.T);
    const Region r = its_uniform(P, C, tab, x);
    return r.item != NONE ? r.item : P.item(r.s);
}

// ---------------------------------------------------------------- selection without replacement
// Collision migration (§4.2): BRS is the method; the naive baselines of Fig. 6(a)
// (repeated sampling) and Fig. 6(b) (updated sampling) exist for the ablation
// of Fig. 10-11.
enum : uint32_t { MIGRATE_BRS = 0, MIGRATE_REPEATED = 1, MIGRATE_UPDATED = 2 };

struct DrawKey {
    uint2 key;       // Philox key (rng_seed)
    uint32_t inst;   // global instance id
    uint32_t t;      // depth
    uint32_t slot;   // frontier vertex id / 0xFFFFFFFF (layer pool)
    uint32_t mode;   // MIGRATE_*
    uint32_t draws;  // accumulated number of draws (statistics, Fig. 11 "#iterations")
};

__device__ __forceinline__ uint64_t wor_draw(const DrawKey& dk, uint32_t j, uint32_t a) {
    return draw_u64(dk.key, dk.inst, dk.t, dk.slot, word3(PURPOSE_EDGE, j, a));
}

__device__ __forceinline__ void bm_set(uint32_t* bm, uint32_t s) {
    atomicOr(bm + (s % BM_WORDS), 1u << (s / BM_WORDS));   // strided mapping (Fig. 7(b))
}
__device__ __forceinline__ bool bm_test(const uint32_t* bm, uint32_t s) {
    return (bm[s % BM_WORDS] >> (s / BM_WORDS)) & 1u;
}

// k distinct picks from pool P; emit(rank, s, item) is called once per pick
// with ranks 0..count-1 in ascending pool-index order (canonical output, R11).
// glist: per-warp global scratch of >= k PickRecs, used only when k > 32.
template <class Pool, class Emit>
__device__ uint32_t select_wor(Pool& P, const Ctps& C, uint64_t* __restrict__ tab, uint32_t* __restrict__ bm,
                               uint32_t k, DrawKey& dk, uint32_t a_max, PickRec* __restrict__ glist,
                               Emit&& emit) {
    const int lane = lane_id();
    const uint32_t n = C.n;
    if (k == 0 || C.npos == 0) return 0;
    if (k >= C.npos) {
        // select all positive-bias candidates, ascending (R8)
        uint32_t rank = 0;
        if constexpr (Pool::kClosedForm) {
            for (uint32_t i0 = 0; i0 < n; i0 += 32) {
                const uint32_t i = i0 + lane;
                if (i < n) emit(rank + lane, i, P.item(i));
                rank += min(32u, n - i0);
            }
        } else if (C.m == 0) {
            for (uint32_t i0 = 0; i0 < n; i0 += 32) {
                const uint32_t i = i0 + lane;
                const bool pos = i < n && tab[i] > (i ? tab[i - 1] : 0);
                const unsigned bal = __ballot_sync(FULL, pos);
                if (pos) emit(rank + __popc(bal & lanemask_lt()), i, P.item(i));
                rank += __popc(bal);
            }
        } else {
            const uint32_t nrows = (n + 31) >> 5;
            P.seek(0);
            for (uint32_t r0 = 0; r0 < nrows; r0 += U) {
                uint32_t key[U], b[U];
                P.template load_rows<U>(r0, key, b);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool pos = b[u] > 0;
                    const unsigned bal = __ballot_sync(FULL, pos);
                    if (pos) emit(rank + __popc(bal & lanemask_lt()), (r0 + u) * 32 + lane, key[u]);
                    rank += __popc(bal);
                }
            }
        }
        return C.npos;
    }

    const bool use_bm = n <= BM_BITS;
    if (use_bm) {
        const uint32_t words = min(n, static_cast<uint32_t>(BM_WORDS));
        for (uint32_t w = lane; w < words; w += 32) bm[w] = 0;
        __syncwarp();
    }
    const uint64_t T = C.T;
    const uint32_t npass = (k + 31) / 32;
    uint32_t fin = NONE, fin_b = 0;
    uint64_t fin_lo = 0;

    for (uint32_t pass = 0; pass < npass; ++pass) {
        const uint32_t j0 = pass * 32;
        const uint32_t kp = min(32u, k - j0);
        const uint32_t nprev = j0;   // picks finalised in earlier passes (in glist / bitmap)
        // taken test against earlier passes
        auto taken_prev = [&](uint32_t s) -> bool {
            if (use_bm) return bm_test(bm, s);
            for (uint32_t q = 0; q < nprev; ++q)
                if (glist[q].s == s) return true;
            return false;
        };
        // ---- attempt 0 for every lane of the pass (one lane per pick)
        Region reg;
        reg.s = NONE; reg.b = 0; reg.lo = 0; reg.item = NONE;
        const bool updated_mode = dk.mode == MIGRATE_UPDATED;
        if (!updated_mode) {
            const uint64_t x0 = below(wor_draw(dk, j0 + lane, 0), T);
            dk.draws += kp;
            if constexpr (Pool::kClosedForm) {
                reg.s = static_cast<uint32_t>(x0); reg.lo = x0; reg.b = 1;
            } else if (C.m == 0) {
                if (static_cast<uint32_t>(lane) < kp) reg = its_table(tab, n, x0);
            } else {
                for (uint32_t l = 0; l < kp; ++l) {
                    const uint64_t xl = __shfl_sync(FULL, x0, l);
                    const Region rl = its_uniform(P, C, tab, xl);
                    if (static_cast<uint32_t>(lane) == l) reg = rl;
                }
            }
        }
        // updated sampling: no independent attempt-0 candidates (every pick depends
        // on the survivors), so every lane resolves serially below
        uint32_t cand = (static_cast<uint32_t>(lane) < kp && !updated_mode) ? reg.s : NONE;
        fin = NONE; fin_b = 0; fin_lo = 0;

        uint32_t r = 0;   // lanes [0, r) are final
        while (r < kp) {
            const bool active = static_cast<uint32_t>(lane) >= r && static_cast<uint32_t>(lane) < kp;
            const uint32_t v = static_cast<uint32_t>(lane) < r ? fin : (active ? cand : (NONE - lane));
            const unsigned peers = __match_any_sync(FULL, v);
            const unsigned below_r = (r >= 32) ? FULL : ((1u << r) - 1u);
            bool bad = updated_mode && active;
            if (active && !updated_mode) {
                bad = (peers & below_r) != 0                          // equals a final of this pass
                      || (peers & lanemask_lt() & ~below_r) != 0      // same candidate as an earlier open lane
                      || taken_prev(cand);                            // taken in an earlier pass
            }
            const unsigned badm = __ballot_sync(FULL, bad);
            const uint32_t mfirst = badm ? static_cast<uint32_t>(__ffs(badm) - 1) : kp;
            if (static_cast<uint32_t>(lane) >= r && static_cast<uint32_t>(lane) < mfirst) {
                fin = cand; fin_b = reg.b; fin_lo = reg.lo;
                if (use_bm) bm_set(bm, cand);
            }
            __syncwarp();
            r = mfirst;
            if (r >= kp) break;
            // ---- lane r collided with a taken pick: bipartite region search, serially
            const uint32_t jr = j0 + r;
            uint32_t s = __shfl_sync(FULL, reg.s, r);
            uint32_t sb = __shfl_sync(FULL, reg.b, r);
            uint64_t slo = __shfl_sync(FULL, reg.lo, r);
            const uint32_t rr = r;
            auto taken = [&](uint32_t q) -> bool {   // q warp-uniform
                if (use_bm) return bm_test(bm, q);
                if (__ballot_sync(FULL, static_cast<uint32_t>(lane) < rr && fin == q)) return true;
                return taken_prev(q);
            };
            // exact updated sampling over the survivors (Fig. 6(b)) with draw U(jr, aidx):
            // survivor position xs, mapped back to the original CTPS by skipping the
            // taken regions (least fixpoint of y = xs + sum{b_q : taken q, S_q <= y})
            auto updated_pick = [&](uint32_t aidx) -> Region {
                uint64_t tmass = warp_sum(static_cast<uint32_t>(lane) < rr ? fin_b : 0u);
                for (uint32_t q = 0; q < nprev; ++q) tmass += glist[q].b;
                const uint64_t xs = below(wor_draw(dk, jr, aidx), T - tmass);
                uint64_t yy = xs;
                for (;;) {
                    uint64_t add = warp_sum((static_cast<uint32_t>(lane) < rr && fin_lo <= yy) ? fin_b : 0u);
                    for (uint32_t q = 0; q < nprev; ++q)
                        if (glist[q].lo <= yy) add += glist[q].b;
                    const uint64_t ny = xs + add;
                    if (ny == yy) break;
                    yy = ny;
                }
                return its_uniform(P, C, tab, yy);
            };
            Region res;
            uint32_t a = 1;
            if (updated_mode) {
                res = updated_pick(0);
            } else if (dk.mode == MIGRATE_REPEATED) {
                // Fig. 6(a): redraw over the original CTPS until an untaken region is hit
                for (;;) {
                    if (a >= a_max) { res = updated_pick(a_max); ++a; break; }
                    const uint64_t x = below(wor_draw(dk, jr, a), T);
                    ++a;
                    res = its_uniform(P, C, tab, x);
                    if (!taken(res.s)) break;
                }
            } else {
                for (;;) {
                    // (3) fresh draw over the space without [S_s, S_s + b_s); (4)/(5) map back
                    const uint64_t x2 = below(wor_draw(dk, jr, a), T - sb);
                    ++a;
                    const uint64_t y = (x2 < slo) ? x2 : x2 + sb;
                    res = its_uniform(P, C, tab, y);
                    if (!taken(res.s)) break;
                    if (a >= a_max) { res = updated_pick(a_max); ++a; break; }   // R2
                    // (1)(2) plain draw over [0, T)
                    const uint64_t x = below(wor_draw(dk, jr, a), T);
                    ++a;
                    res = its_uniform(P, C, tab, x);
                    if (!taken(res.s)) break;
                    s = res.s; sb = res.b; slo = res.lo;
                }
            }
            dk.draws += updated_mode ? 1u : a - 1u;
            if (static_cast<uint32_t>(lane) == r) {
                fin = res.s; fin_b = res.b; fin_lo = res.lo;
                cand = res.s;
            }
            if (use_bm && lane == 0) bm_set(bm, res.s);
            __syncwarp();
            ++r;
            (void)s;
        }
        if (npass > 1) {
            if (static_cast<uint32_t>(lane) < kp) {
                PickRec pr; pr.s = fin; pr.b = fin_b; pr.lo = fin_lo;
                glist[j0 + lane] = pr;
            }
            __syncwarp();
        }
    }

    // ---- emit in ascending pool order
    if (npass == 1) {
        const uint32_t sorted = warp_sort_u32(fin);
        if (static_cast<uint32_t>(lane) < k) emit(static_cast<uint32_t>(lane), sorted, P.item(sorted));
    } else if (use_bm) {
        uint32_t rank = 0;
        for (uint32_t i0 = 0; i0 < n; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool set = i < n && bm_test(bm, i);
            const unsigned bal = __ballot_sync(FULL, set);
            if (set) emit(rank + __popc(bal & lanemask_lt()), i, P.item(i));
            rank += __popc(bal);
        }
    } else {
        for (uint32_t e = lane; e < k; e += 32) {
            const uint32_t se = glist[e].s;
            uint32_t rank = 0;
            for (uint32_t q = 0; q < k; ++q) rank += glist[q].s < se;
            emit(rank, se, P.item(se));
        }
    }
    return k;
}

// ---------------------------------------------------------------- pools
// N(v) with EdgeBias = deg(u): biased neighbor sampling (Fig. 1) and
// biased DeepWalk.  Rows are 32 consecutive neighbours (one coalesced
// 128 B col load); U rows are loaded before the dependent deg gathers.
struct DegreePool {
    static constexpr bool kClosedForm = false;
    static constexpr bool kCached = false;
    const uint32_t* __restrict__ col;
    const uint32_t* __restrict__ deg;
    uint64_t beg;
    uint32_t n;
    const uint64_t* __restrict__ ccache = nullptr;   // chunk-total cache (rows of d > TAB), optional
    __device__ __forceinline__ void seek(uint32_t) {}
    template <int NR>
    __device__ __forceinline__ void load_rows(uint32_t row0, uint32_t (&key)[NR], uint32_t (&b)[NR]) {
        const int lane = lane_id();
#pragma unroll
        for (int u = 0; u < NR; ++u) {
            const uint32_t i = (row0 + u) * 32 + lane;
            key[u] = (i < n) ? __ldg(col + beg + i) : NONE;
        }
#pragma unroll
        for (int u = 0; u < NR; ++u) b[u] = (key[u] != NONE) ? __ldg(deg + key[u]) : 0u;
    }
    __device__ __forceinline__ uint32_t item(uint32_t i) const { return __ldg(col + beg + i); }
};

// N(v) with EdgeBias = 1: closed form S_i = i -- only the chosen
// col entries are ever read.
struct UniformPool {
    static constexpr bool kClosedForm = true;
    static constexpr bool kCached = false;
    const uint32_t* __restrict__ col;
    uint64_t beg;
    uint32_t n;
    __device__ __forceinline__ void seek(uint32_t) {}
    template <int NR>
    __device__ __forceinline__ void load_rows(uint32_t row0, uint32_t (&key)[NR], uint32_t (&b)[NR]) {
        const int lane = lane_id();
#pragma unroll
        for (int u = 0; u < NR; ++u) {
            const uint32_t i = (row0 + u) * 32 + lane;
            key[u] = (i < n) ? __ldg(col + beg + i) : NONE;
            b[u] = i < n ? 1u : 0u;
        }
    }
    __device__ __forceinline__ uint32_t item(uint32_t i) const { return __ldg(col + beg + i); }
};

// ---------------------------------------------------------------- CTPS-cache B-tree
// Static fanout-32 index over one row's cached inclusive prefix cps[beg, beg+d):
// level 0 = the row itself; level k+1 entry j = max of level-k block j (its last
// entry); levels until <= 32 entries.  Stored top level first at bt[boff...].
// A search reads one coalesced 32-entry block per level (256 B) instead of 32
// scattered probes, and the top level's last entry is T.
struct CpsTree {
    const uint64_t* __restrict__ cps;
    const uint64_t* __restrict__ bt;
    const uint32_t* __restrict__ col;
    uint64_t beg;
    uint32_t d;
    uint64_t boff;

    // levels: n_k = ceil(d / 32^k) entries at level k; K = first k with n_k <= 32
    // (closed form, no per-step loop over arrays).
    __device__ __forceinline__ static int num_levels(uint32_t d) {
        return d <= 32 ? 0 : (31 - __clz(d - 1)) / 5;   // (bits(d-1) - 1) / 5
    }
    // Warp-collective.  kDraw: x = below(U, T) with T from the top level (returned);
    // else x is given.  Result: CSR index e of the pick, S_s = lo, S_{s+1} = hi, col[e].
    template <bool kDraw, bool kMeta = false>
    __device__ __forceinline__ void search(uint64_t U, uint64_t& x, uint64_t& T, uint64_t& e, uint64_t& lo,
                                           uint64_t& hi, uint32_t& item, uint32_t& probes,
                                           const uint64_t* __restrict__ nmp = nullptr, uint64_t* meta = nullptr) const {
        const int lane = lane_id();
        const int K = num_levels(d);
        uint32_t j = 0;          // block index at the current level
        uint64_t left = 0;       // S just left of the current block
        uint64_t off = 0;        // offset of level k inside the row's bt segment (top level first)
        for (int k = K; k >= 0; --k) {
            const uint32_t nk = k == 0 ? d : ((d - 1) >> (5 * k)) + 1;
            const uint32_t idx = j * 32 + lane;
            const bool valid = idx < nk;
            uint64_t v = 0, mt = 0;
            uint32_t it = NONE;
            if (valid) {
                if (k == 0) {
                    v = __ldg(cps + beg + idx);
                    it = __ldg(col + beg + idx);
                    if constexpr (kMeta) mt = __ldg(nmp + beg + idx);   // next vertex's (row_ptr, degree)
                }
                else v = __ldg(bt + boff + off + idx);
            }
            probes += min(32u, nk - j * 32);
            if (kDraw && k == K) {   // top level: its last entry is the row total
                T = __shfl_sync(FULL, v, nk - 1);
                if (T == 0) { e = ~0ull; item = NONE; lo = hi = 0; return; }
                x = below(U, T);
            }
            const unsigned hit = __ballot_sync(FULL, valid && v > x);
            const int f = __ffs(hit) - 1;   // exists for x < T
            const uint64_t pv = __shfl_sync(FULL, v, f > 0 ? f - 1 : 0);
            if (f > 0) left = pv;
            if (k == 0) {
                e = beg + idx - lane + f;
                hi = __shfl_sync(FULL, v, f);
                lo = left;
                item = __shfl_sync(FULL, it, f);
                if constexpr (kMeta) *meta = __shfl_sync(FULL, mt, f);
            }
            off += nk;
            j = j * 32 + f;
        }
    }
};

// N(v) with EdgeBias = deg(u) read from the static-bias CTPS cache (P:779-789,
// reading R25): cps[beg + i] = S_{i+1}.  T is one load; a draw is located by a
// 32-ary warp search of the cached prefix (O(log32 d) round trips) -- the same
// integer S as DegreePool's scan, hence the same picks.
// The narrow walk index's vertex heads (wix.cuh), when built with leaf fanout 128: cached
// degree selections search them (head -> (node) -> leaf) instead of the u64 B-tree.
struct WixPtrs {
    const uint32_t* head = nullptr;
    const uint32_t* c32 = nullptr;
    const uint32_t* col = nullptr;
    const uint32_t* inn = nullptr;
};

struct CachedDegreePool {
    static constexpr bool kClosedForm = false;
    static constexpr bool kCached = true;
    const uint32_t* __restrict__ col;
    const uint64_t* __restrict__ cps;
    uint64_t beg;
    uint32_t n;
    uint32_t np;          // positive-bias candidates of the row
    uint32_t probes;      // cache loads issued (statistics)
    const uint64_t* __restrict__ bt;   // B-tree index (CpsTree)
    uint64_t boff;
    WixPtrs wx{};                      // vertex heads (optional)
    uint32_t vid = 0;                  // the pool's vertex (head address)
    __device__ __forceinline__ uint64_t total() const { return n ? __ldg(cps + beg + n - 1) : 0; }
    __device__ __forceinline__ uint32_t npos_count() const { return np; }
    __device__ __forceinline__ Region search(uint64_t x) {
        if (wx.head) {   // T < 2^32 for every row when the heads exist
            uint32_t s, lo, b, it, nb;
            wix_head_search<128>(wx.head, wx.c32, wx.col, wx.inn, vid, static_cast<uint32_t>(x), s, lo, b, it, nb);
            probes += nb / 8;   // in 8 B cache-entry units (statistics)
            Region r;
            r.s = s; r.lo = lo; r.b = b; r.item = it;
            return r;
        }
        CpsTree t{cps, bt, col, beg, n, boff};
        uint64_t T = 0, e = 0, lo = 0, hi = 0;
        uint32_t item = NONE;
        t.template search<false>(0, x, T, e, lo, hi, item, probes);
        Region r;
        r.s = static_cast<uint32_t>(e - beg);
        r.lo = lo;
        r.b = static_cast<uint32_t>(hi - lo);
        r.item = item;
        return r;
    }
    __device__ __forceinline__ void seek(uint32_t) {}
    template <int NR>
    __device__ __forceinline__ void load_rows(uint32_t row0, uint32_t (&key)[NR], uint32_t (&b)[NR]) {
        const int lane = lane_id();
#pragma unroll
        for (int u = 0; u < NR; ++u) {
            const uint32_t i = (row0 + u) * 32 + lane;
            key[u] = NONE;
            b[u] = 0;
            if (i < n) {
                key[u] = __ldg(col + beg + i);
                const uint64_t prev = i ? __ldg(cps + beg + i - 1) : 0;
                b[u] = static_cast<uint32_t>(__ldg(cps + beg + i) - prev);
            }
        }
    }
    __device__ __forceinline__ uint32_t item(uint32_t i) const { return __ldg(col + beg + i); }
};

}  // namespace csaw
