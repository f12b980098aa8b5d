// n2v_index.cu — node2vec per-edge intersection index (CSAW_GRAPH_N2V_INDEX) and the
// thread-per-walker node2vec kernel that searches it.
//
// A node2vec step at v arriving from prev (R16) selects from N(v) with the
// integer biases wp (u == prev), w1 (u in N(prev)), wq (otherwise).  Its CTPS is
// piecewise linear: S grows by wq per position except at the "specials" -- prev
// itself and the common neighbours N(v) ∩ N(prev).  For a member at position p of
// N(v) with j members before it,
//     S(p) = wq p - (wq - w1) j - (wq - wp) [p > ppos]          (ppos = position of prev),
// so the region of a draw x follows from the LAST special with S <= x and a closed
// form between specials (the same algebra as k_node2vec_tri's n2t_specials).
//
// The specials depend only on the directed edge e = (prev -> v) -- a static property
// of the graph, for any p and q -- so they are listed once per edge at graph creation
// (the paper's deleted "caching transition probability", R25, applied to
// the dynamic node2vec bias keyed by the edge the walker arrived by):
//     rec[e] (128 B; N2X_P = 24) = {index offset (40 bits) | C = |N(v) ∩ N(prev)| (24 bits),
//                      ppos, mb, v = col[e], row start of v (40 bits) | deg(v) (24 bits), 0,
//                      P[0..cap)}
//         mb = members before ppos (members with value < prev: rows are sorted)
//         cap = 48 u16 values when deg(v) <= 65,536 (every position fits 16 bits), else 24 u32
//         P  = the member positions themselves when C <= cap, else cap splitters
//              P[k] = I[j_k], j_k = floor((k + 1) C / (cap + 1))
//     idx[off ..) = ascending positions I in N(v) of the members (C > cap only; u16 for narrow rows).
// The record of the entry a walker arrived by carries everything the next step needs
// (its vertex, row and degree, and the step's specials or their splitters), so a step
// is one record and, for C > N2X_P, a binary search of about log2(C / (N2X_P + 1)) probes
// between two splitters: O(log C) dependent sectors instead of a merge of N(v) with
// N(prev).  The pick is bit-identical to the full CTPS (same integer S, same draw) and
// to the oracle.  Record size: a random read moves a whole 128 B line from HBM whether 64 or
// 128 B are asked for (profiles/r02_random_granule.txt, r3k TMA measurement), so 128 B
// records hold 24 inline values for the DRAM cost of 8 (A/B cfg3: 6.21 vs 6.97 ms).
// Memory: 128 B per CSR entry + 4 B per (edge, common neighbour) pair of the edges with
// C > N2X_P; built only if it fits (best-effort).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "util.cuh"


namespace csaw {

// Inline area of a record (96 B): the member positions / splitters in N(v) as 2 N2X_P u16 values
// when every position of N(v) fits 16 bits (deg(v) <= 65,536: "narrow"), else N2X_P u32 values.
#ifndef N2X_NARROW_DEG_N
#define N2X_NARROW_DEG_N 65536   // 0: u32 inline values only (A/B)
#endif
constexpr uint32_t N2X_NARROW_DEG = N2X_NARROW_DEG_N;
__host__ __device__ __forceinline__ bool n2x_narrow(uint64_t d) { return d <= N2X_NARROW_DEG; }
__host__ __device__ __forceinline__ uint32_t n2x_cap(uint64_t d) { return n2x_narrow(d) ? 2 * N2X_P : N2X_P; }
__device__ __forceinline__ uint32_t n2x_get(const void* P, bool narrow, uint32_t k) {
    return narrow ? static_cast<uint32_t>(static_cast<const uint16_t*>(P)[k]) : static_cast<const uint32_t*>(P)[k];
}
__device__ __forceinline__ void n2x_put(void* P, bool narrow, uint32_t k, uint32_t v) {
    if (narrow) static_cast<uint16_t*>(P)[k] = static_cast<uint16_t>(v);
    else static_cast<uint32_t*>(P)[k] = v;
}
// rank of splitter k of C members: floor((k + 1) C / (cap + 1)), cap = 48 or 24 ((k + 1) C < 2^30)
__host__ __device__ __forceinline__ uint32_t n2x_split(bool narrow, uint32_t k, uint32_t C) {
    return narrow ? ((k + 1) * C) / (2 * N2X_P + 1) : ((k + 1) * C) / (N2X_P + 1);
}

// ---------------------------------------------------------------- build
// Hub rank bitmaps: for the vertices of highest degree (d >= N2X_HUB_DEG, up to a memory
// cap) a bitmap of N(h) over [0, V) plus the count of set bits before every 512-bit block.
// Intersecting a list with a hub's list then costs one bit test per element (membership)
// and a popcount over one 64 B line (its position in N(h)) instead of a binary search of
// the hub's row -- the hub-hub pairs dominate the build.
#ifndef N2X_HUB_DEG
#define N2X_HUB_DEG 1024
#endif
#ifndef N2X_HUB_MAX_BYTES
#define N2X_HUB_MAX_BYTES (4ull << 30)   // bitmap scratch during the build
#endif
struct HubRank {
    const int32_t* __restrict__ hid;       // [V] hub slot or -1 (nullptr: no hubs)
    const uint64_t* __restrict__ bits;     // [nhub][W]
    const uint32_t* __restrict__ bcnt;     // [nhub][W / 8 + 1]
    uint64_t W;                            // words per bitmap (multiple of 8)
    // position of x in N(h) if x is a member
    __device__ __forceinline__ bool find(int32_t h, uint32_t x, uint64_t& pos) const {
        const uint64_t* b = bits + static_cast<uint64_t>(h) * W;
        const uint64_t wi = x >> 6;
        const uint64_t w = __ldg(b + wi);
        if (!((w >> (x & 63)) & 1ull)) return false;
        const uint64_t blk = wi >> 3;
        uint64_t c = __ldg(bcnt + static_cast<uint64_t>(h) * (W / 8 + 1) + blk);
        for (uint64_t k = blk * 8; k < wi; ++k) c += __popcll(__ldg(b + k));
        pos = c + __popcll(w & ((1ull << (x & 63)) - 1ull));
        return true;
    }
};

__global__ void k_hub_bits(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                           const uint32_t* __restrict__ hubs, uint32_t nhub, uint64_t W, uint64_t* __restrict__ bits) {
    for (uint32_t h = blockIdx.x; h < nhub; h += gridDim.x) {
        const uint32_t v = hubs[h];
        uint64_t* b = bits + static_cast<uint64_t>(h) * W;
        for (int64_t e = rp[v] + threadIdx.x; e < rp[v + 1]; e += blockDim.x) {
            const uint32_t x = col[e];
            atomicOr(reinterpret_cast<unsigned long long*>(b + (x >> 6)), 1ull << (x & 63));
        }
    }
}

// bcnt[h][k] = set bits of words [0, 8 k): one block per hub, a block scan of block counts
template <int NT>
__global__ void k_hub_cnt(const uint64_t* __restrict__ bits, uint32_t nhub, uint64_t W, uint32_t* __restrict__ bcnt) {
    __shared__ uint64_t wsum[NT / 32];
    __shared__ uint64_t total;
    const uint64_t nb = W / 8;
    for (uint32_t h = blockIdx.x; h < nhub; h += gridDim.x) {
        const uint64_t* b = bits + static_cast<uint64_t>(h) * W;
        uint32_t* c = bcnt + static_cast<uint64_t>(h) * (nb + 1);
        const uint64_t per = (nb + NT - 1) / NT;
        const uint64_t k0 = min(nb, threadIdx.x * per), k1 = min(nb, k0 + per);
        uint64_t s = 0;
        for (uint64_t k = k0; k < k1; ++k)
            for (int j = 0; j < 8; ++j) s += __popcll(b[8 * k + j]);
        uint64_t run = block_excl_scan<NT>(s, wsum, &total);
        for (uint64_t k = k0; k < k1; ++k) {
            c[k] = static_cast<uint32_t>(run);
            for (int j = 0; j < 8; ++j) run += __popcll(b[8 * k + j]);
        }
        if (threadIdx.x == 0) c[nb] = static_cast<uint32_t>(total);
        __syncthreads();
    }
}

// One warp per undirected edge {v, u} (entry e = (v -> u) with u > v, its reverse r =
// (u -> v)).  The shorter list is walked in rows of 32; each entry's lower bound in the
// longer list gives its position there.  Pass 1 (kList = false) writes the records'
// C, ppos and mb; pass 2 lists the member positions into both edges' index ranges.
// Edges are handed out in chunks of N2X_BUILD_CHUNK from a global ticket (hub-hub pairs cost
// far more than the rest; a static split leaves a few warps with the heavy tail).
#ifndef N2X_BUILD_CHUNK
#define N2X_BUILD_CHUNK 16
#endif
template <bool kList>
__global__ void k_n2x(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                      const uint32_t* __restrict__ src, int64_t E, uint4* __restrict__ rec,
                      uint32_t* __restrict__ idx, unsigned int* __restrict__ asym, HubRank hr,
                      unsigned long long* __restrict__ ticket) {
    const int lane = lane_id();
    uint64_t e = 0, chunk_end = 0;
    for (;;) {
        if (e >= chunk_end) {
            unsigned long long t0 = 0;
            if (lane == 0) t0 = atomicAdd(ticket, static_cast<unsigned long long>(N2X_BUILD_CHUNK));
            e = __shfl_sync(FULL, t0, 0);
            chunk_end = e + N2X_BUILD_CHUNK;
        }
        if (e >= static_cast<uint64_t>(E)) break;
        const uint64_t ecur = e++;
        const uint32_t v = src[ecur], u = col[ecur];
        if (u == v) { if (lane == 0) atomicOr(asym, 1u); continue; }
        if (u < v) continue;
        const int64_t bv = rp[v], bu = rp[u];
        const uint64_t dv = static_cast<uint64_t>(rp[v + 1] - bv), du = static_cast<uint64_t>(rp[u + 1] - bu);
        const uint64_t j = warp_lower_bound(col + bu, 0, du, v);   // position of v in N(u)
        if (!(j < du && __ldg(col + bu + j) == v)) { if (lane == 0) atomicOr(asym, 1u); continue; }
        const uint64_t r = static_cast<uint64_t>(bu) + j;
        const bool sv = dv <= du;                                   // N(v) is the shorter list
        const uint32_t* small = col + (sv ? bv : bu);
        const uint32_t* big = col + (sv ? bu : bv);
        const uint64_t ns = sv ? dv : du, nb = sv ? du : dv;
        uint64_t off_e = 0, off_r = 0;
        uint32_t C_all = 0;
        if (kList) {
            const uint4 re = rec[N2X_U4 * ecur], rr = rec[N2X_U4 * r];
            off_e = re.x | (static_cast<uint64_t>(re.y & 0xFFu) << 32);
            off_r = rr.x | (static_cast<uint64_t>(rr.y & 0xFFu) << 32);
            C_all = re.y >> 8;
        }
        uint32_t cnt = 0, below_v = 0, below_u = 0;
        uint64_t lo0 = 0;
        const int32_t hb = hr.hid ? __ldg(hr.hid + (sv ? u : v)) : -1;   // the longer list's owner a hub?
        for (uint64_t r0 = 0; r0 < ns && lo0 < nb; r0 += 32) {
            const uint64_t i = r0 + lane;
            const bool valid = i < ns;
            const uint32_t x = valid ? __ldg(small + i) : NONE;
            uint64_t l = 0, hi = 0;
            bool f;
            if (hb >= 0) {   // bit test + rank in the hub's bitmap
                f = valid && hr.find(hb, x, l);
            } else {
                const uint32_t xmin = __shfl_sync(FULL, x, 0);
                const int last = static_cast<int>(ns - 1 - r0 < 31 ? ns - 1 - r0 : 31);
                const uint32_t xmax = __shfl_sync(FULL, x, last);
                const uint64_t lo = warp_lower_bound(big, lo0, nb, xmin);
                hi = xmax == NONE ? nb : warp_lower_bound(big, lo, nb, xmax + 1u);
                l = lo;
                uint64_t h = hi;
                while (l < h) {   // same trip count on every lane
                    const uint64_t mid = (l + h) >> 1;
                    if (__ldg(big + mid) < x) l = mid + 1; else h = mid;
                }
                f = valid && l < hi && __ldg(big + l) == x;
            }
            const unsigned m = __ballot_sync(FULL, f);
            if (kList) {
                if (f) {
                    const uint32_t rank = cnt + __popc(m & lanemask_lt());
                    const uint32_t pu = static_cast<uint32_t>(sv ? l : i), pv = static_cast<uint32_t>(sv ? i : l);
                    // entry e (walker at u): positions in N(u); entry r (walker at v): positions in N(v);
                    // listed in idx when C exceeds that record's inline capacity, else inline
                    n2x_put(C_all > n2x_cap(du) ? static_cast<void*>(idx + off_e) : static_cast<void*>(rec + N2X_U4 * ecur + 2),
                            n2x_narrow(du), rank, pu);
                    n2x_put(C_all > n2x_cap(dv) ? static_cast<void*>(idx + off_r) : static_cast<void*>(rec + N2X_U4 * r + 2),
                            n2x_narrow(dv), rank, pv);
                }
            } else {
                below_v += __popc(__ballot_sync(FULL, f && x < v));
                below_u += __popc(__ballot_sync(FULL, f && x < u));
            }
            cnt += __popc(m);
            if (hb < 0) lo0 = hi;
        }
        if (!kList && lane == 0) {
            // e = (v -> u): a walker at u that came from v; prev = v sits at position j of N(u)
            rec[N2X_U4 * ecur] = make_uint4(0u, cnt << 8, static_cast<uint32_t>(j), below_v);
            // r = (u -> v): a walker at v that came from u; prev = u sits at position e - bv of N(v)
            rec[N2X_U4 * r] = make_uint4(0u, cnt << 8, static_cast<uint32_t>(ecur - static_cast<uint64_t>(bv)), below_u);
        }
    }
}

// exclusive scan of the listed member counts (C > N2X_P) into the records' 40-bit offsets
struct N2xCount {
    const uint4* rec;
    const int64_t* rp;
    const uint32_t* col;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
        const uint32_t c = rec[N2X_U4 * i].y >> 8;
        const uint32_t v = col[i];
        const uint64_t d = static_cast<uint64_t>(rp[v + 1] - rp[v]);
        return c > n2x_cap(d) ? (n2x_narrow(d) ? (c + 1) / 2 : c) : 0;   // u32 units (narrow rows: u16 pairs)
    }
};
struct N2xOffset {
    uint4* rec;
    unsigned long long* sum;
    __device__ __forceinline__ void operator()(uint64_t i, uint64_t e, uint64_t) const {
        rec[N2X_U4 * i].x = static_cast<uint32_t>(e);
        rec[N2X_U4 * i].y = static_cast<uint32_t>(e >> 32) | (rec[N2X_U4 * i].y & 0xFFFFFF00u);
    }
    __device__ __forceinline__ void total(uint64_t, uint64_t t) const { *sum = t; }
};

// rest of each record: the entry's vertex v = col[e], its row start and degree, and for
// C > N2X_P the N2X_P splitters P[k] = I[floor((k + 1) C / (N2X_P + 1))] (C <= N2X_P: the list pass
// wrote P)
__global__ void k_n2x_dst(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col, int64_t E,
                          const uint32_t* __restrict__ idx, uint4* __restrict__ rec) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = col[e];
        const uint64_t rs = static_cast<uint64_t>(rp[v]);
        const uint32_t d = static_cast<uint32_t>(rp[v + 1] - rp[v]);
        rec[N2X_U4 * e + 1] = make_uint4(v, static_cast<uint32_t>(rs), static_cast<uint32_t>(rs >> 32) | (d << 8), 0u);
        const uint4 q = rec[N2X_U4 * e];
        const uint32_t C = q.y >> 8;
        const bool nw = n2x_narrow(d);
        const uint32_t cap = n2x_cap(d);
        if (C > cap) {
            const uint32_t* I = idx + (q.x | (static_cast<uint64_t>(q.y & 0xFFu) << 32));
            void* P = rec + N2X_U4 * e + 2;
            for (uint32_t k = 0; k < cap; ++k) n2x_put(P, nw, k, n2x_get(I, nw, n2x_split(nw, k, C)));
        }
    }
}

__global__ void k_n2x_src(const int64_t* __restrict__ rp, int64_t V, uint32_t* __restrict__ src) {
    const int lane = lane_id();
    for (uint64_t v = global_warp_id(); v < static_cast<uint64_t>(V); v += total_warps())
        for (int64_t e = rp[v] + lane; e < rp[v + 1]; e += 32) src[e] = static_cast<uint32_t>(v);
}

csaw_status build_n2v_index(csaw_graph* g, int blocks) {
    if (!g->rows_sorted || g->E <= 0 || g->max_deg >= (int64_t(1) << 24)) return CSAW_OK;
    const int64_t E = g->E;
    uint32_t* src = nullptr;
    unsigned int* asym = nullptr;
    unsigned long long* tot = nullptr;
    uint64_t* part = nullptr;
    auto release = [&]() {
        if (src) cudaFree(src);
        if (asym) cudaFree(asym);
        if (tot) cudaFree(tot);
        if (part) cudaFree(part);
        cudaGetLastError();
    };
    auto drop = [&]() {   // best-effort: without the index node2vec uses k_node2vec_tri / the merge kernel
        release();
        if (g->n2x_rec) cudaFree(g->n2x_rec);
        if (g->n2x_idx) cudaFree(g->n2x_idx);
        g->n2x_rec = nullptr;
        g->n2x_idx = nullptr;
        g->n2x_total = 0;
        cudaGetLastError();
        return CSAW_OK;
    };
    if (cudaMalloc(&src, sizeof(uint32_t) * E) != cudaSuccess || cudaMalloc(&asym, sizeof(unsigned int)) != cudaSuccess ||
        cudaMalloc(&tot, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&part, sizeof(uint64_t) * (SCAN_MAX_GRID + 8)) != cudaSuccess ||
        cudaMalloc(&g->n2x_rec, N2X_U4 * sizeof(uint4) * E) != cudaSuccess)
        return drop();
    if (g->E >= (int64_t(1) << 40)) return drop();
    cudaMemset(asym, 0, sizeof(unsigned int));
    cudaMemset(tot, 0, sizeof(unsigned long long));          // the count pass's edge ticket
    cudaMemset(g->n2x_rec, 0xFF, N2X_U4 * sizeof(uint4) * E);   // unused inline slots
    k_n2x_src<<<blocks, 256>>>(g->row_ptr, g->V, src);
    // hub rank bitmaps for the highest-degree rows (build scratch, freed below): at most
    // N2X_HUB_MAX_BYTES, the largest degrees first
    HubRank hr{nullptr, nullptr, nullptr, 0};
    int32_t* hid = nullptr;
    uint32_t* hubs = nullptr;
    uint64_t* hbits = nullptr;
    uint32_t* hcnt = nullptr;
    auto free_hubs = [&]() {
        if (hid) cudaFree(hid);
        if (hubs) cudaFree(hubs);
        if (hbits) cudaFree(hbits);
        if (hcnt) cudaFree(hcnt);
        hid = nullptr; hubs = nullptr; hbits = nullptr; hcnt = nullptr;
        cudaGetLastError();
    };
    {
        std::vector<int64_t> hrp(static_cast<size_t>(g->V) + 1);
        std::vector<uint32_t> hv;
        if (cudaMemcpy(hrp.data(), g->row_ptr, sizeof(int64_t) * (g->V + 1), cudaMemcpyDeviceToHost) == cudaSuccess) {
            for (int64_t v = 0; v < g->V; ++v)
                if (hrp[v + 1] - hrp[v] >= N2X_HUB_DEG) hv.push_back(static_cast<uint32_t>(v));
            std::sort(hv.begin(), hv.end(), [&](uint32_t a, uint32_t b) {
                return hrp[a + 1] - hrp[a] > hrp[b + 1] - hrp[b];
            });
            const uint64_t W = ((static_cast<uint64_t>(g->V) + 63) / 64 + 7) / 8 * 8;
            const uint64_t per = W * 8 + (W / 8 + 1) * 4;
            const uint64_t cap = static_cast<uint64_t>(N2X_HUB_MAX_BYTES) / per;
            if (hv.size() > cap) hv.resize(cap);
            const uint32_t nhub = static_cast<uint32_t>(hv.size());
            std::vector<int32_t> hh(static_cast<size_t>(g->V), -1);
            for (uint32_t k = 0; k < nhub; ++k) hh[hv[k]] = static_cast<int32_t>(k);
            if (nhub > 0 && cudaMalloc(&hid, sizeof(int32_t) * g->V) == cudaSuccess &&
                cudaMalloc(&hubs, sizeof(uint32_t) * nhub) == cudaSuccess &&
                cudaMalloc(&hbits, sizeof(uint64_t) * W * nhub) == cudaSuccess &&
                cudaMalloc(&hcnt, sizeof(uint32_t) * (W / 8 + 1) * nhub) == cudaSuccess) {
                cudaMemcpy(hid, hh.data(), sizeof(int32_t) * g->V, cudaMemcpyHostToDevice);
                cudaMemcpy(hubs, hv.data(), sizeof(uint32_t) * nhub, cudaMemcpyHostToDevice);
                cudaMemset(hbits, 0, sizeof(uint64_t) * W * nhub);
                k_hub_bits<<<std::min<uint32_t>(nhub, 65535), 256>>>(g->row_ptr, g->col, hubs, nhub, W, hbits);
                k_hub_cnt<256><<<std::min<uint32_t>(nhub, 65535), 256>>>(hbits, nhub, W, hcnt);
                hr = HubRank{hid, hbits, hcnt, W};
            } else {
                free_hubs();   // an accelerator of the build: without it, binary searches
            }
        }
    }
    k_n2x<false><<<blocks * 4, 256>>>(g->row_ptr, g->col, src, E, g->n2x_rec, nullptr, asym, hr, tot);
    unsigned int h = 0;
    if (cudaMemcpy(&h, asym, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess || h)   // not symmetric
        return (free_hubs(), drop());
    if (device_scan(N2xCount{g->n2x_rec, g->row_ptr, g->col}, static_cast<uint64_t>(E), N2xOffset{g->n2x_rec, tot}, part, nullptr) != CSAW_OK)
        return (free_hubs(), drop());
    unsigned long long total = 0;
    if (cudaMemcpy(&total, tot, sizeof(total), cudaMemcpyDeviceToHost) != cudaSuccess) return (free_hubs(), drop());
    if (total >= (1ull << 40)) return (free_hubs(), drop());
    // + 8 entries: a search reads whole 32 B groups of member positions (N2X_SECTOR_PROBES)
    if (cudaMalloc(&g->n2x_idx, sizeof(uint32_t) * (total + 8)) != cudaSuccess) return (free_hubs(), drop());
    cudaMemset(g->n2x_idx + total, 0, sizeof(uint32_t) * 8);
    g->n2x_total = total;
    cudaMemset(tot, 0, sizeof(unsigned long long));   // the list pass's edge ticket (the scan total was read)
    k_n2x<true><<<blocks * 4, 256>>>(g->row_ptr, g->col, src, E, g->n2x_rec, g->n2x_idx, asym, hr, tot);
    k_n2x_dst<<<blocks * 4, 256>>>(g->row_ptr, g->col, E, g->n2x_idx, g->n2x_rec);
    const cudaError_t se = cudaDeviceSynchronize();
    free_hubs();
    if (se != cudaSuccess) return drop();
    release();
    return CSAW_OK;
}

// ---------------------------------------------------------------- walk
struct N2xArgs {
    const int64_t* __restrict__ rp;
    const uint4* __restrict__ rec;            // [N2X_U4 E]: 16 N2X_U4 B per entry
    const uint32_t* __restrict__ idx;
    uint64_t idx_n;                           // u32 units of idx (debug bounds checks)
    const uint32_t* __restrict__ seeds;
    uint64_t n;
    int32_t L;
    uint32_t base;
    uint2 key;
    uint32_t* __restrict__ path;
    unsigned long long* __restrict__ counters;   // [1] steps, [2] index probes, [3] sector bytes, [7] group ticket
    uint32_t wp, w1, wq;    // integer biases (R16), each < 2^30 (checked by the launcher)
    int32_t wq_shift;       // log2(wq) if wq is a power of two, else -1
    double wq_inv;          // 1 / wq (quotients of dividends < 2^53, corrected by one step)
};

// floor(a / wq) for 0 <= a < 2^53 without the 64-bit division subroutine: a shift when wq is a
// power of two (p = 2, q = 0.5 gives wq = 4), else a double-precision estimate corrected by one
__device__ __forceinline__ uint32_t n2x_div(int64_t a, const N2xArgs& A) {
    if (A.wq_shift >= 0) return static_cast<uint32_t>(a >> A.wq_shift);
    int64_t q = static_cast<int64_t>(static_cast<double>(a) * A.wq_inv);
    const int64_t r = a - q * static_cast<int64_t>(A.wq);
    if (r < 0) --q;
    else if (r >= static_cast<int64_t>(A.wq)) ++q;
    return static_cast<uint32_t>(q);
}

// S(j, p) = wq p - dq1 j - sub, exact in int64 (wq < 2^32, p, j < 2^24; dq1 may be negative):
// the CTPS at the member of rank j and position p (sub = wq - wp after prev, else 0)
__device__ __forceinline__ int64_t n2x_S(uint32_t wq, int64_t dq1, uint32_t p, uint32_t j, int64_t sub) {
    // |dq1| < 2^30 and j < 2^24: 32 x 32 -> 64-bit products (IMAD.WIDE), no 64-bit multiply
    return static_cast<int64_t>(static_cast<uint64_t>(wq) * p) -
           static_cast<int64_t>(static_cast<int32_t>(dq1)) * static_cast<int64_t>(static_cast<int32_t>(j)) - sub;
}

// Narrow the member-rank range [lo, hi) of the draw x with the record's N2X_P inline values P:
// the member positions themselves when C <= N2X_P (then [l, h) is resolved: h = l), else
// splitters at ranks j_k = floor((k + 1) C / (N2X_P + 1)).  The predicate "j_k < lo, or j_k < hi
// and S(j_k, P[k]) <= x" holds on a prefix of k (S increases with the rank), so a binary search
// over k reads about log2(N2X_P) inline values.  On return l - 1 is the last rank known to pass
// (pos = its position if l > lo) and h the first known to fail.
__device__ __forceinline__ void n2x_inline(const void* P, bool narrow, uint32_t C, uint32_t lo, uint32_t hi,
                                           int64_t x, uint32_t wq, int64_t dq1, int64_t sub, uint32_t& l, uint32_t& h,
                                           uint32_t& pos) {
    const uint32_t cap = narrow ? 2 * N2X_P : N2X_P;
    const bool in = C <= cap;
    uint32_t a0 = 0, a1 = in ? C : cap;
    l = lo;
    h = hi;
    while (a0 < a1) {
        const uint32_t k = (a0 + a1) >> 1;
        const uint32_t j = in ? k : n2x_split(narrow, k, C);
        bool t = j < lo;
        if (!t && j < hi) {
            const uint32_t pk = n2x_get(P, narrow, k);
            t = n2x_S(wq, dq1, pk, j, sub) <= x;
            if (t) { l = j + 1; pos = pk; } else h = j;
        }
        if (t) a0 = k + 1; else a1 = k;
    }
    if (in) h = l;
}

// Last member rank j in [lo, hi) with S(j, I[j]) <= x; found = false if none, else pos = I[j]:
// the inline values, then a plain binary search over idx between two splitters (about
// log2(C / (N2X_P + 1)) probes).
__device__ __forceinline__ uint32_t n2x_last_le(const uint32_t* __restrict__ I, const void* P, bool narrow,
                                                uint32_t C, uint32_t lo, uint32_t hi, int64_t x, uint32_t wq,
                                                int64_t dq1, int64_t sub, uint32_t& probes, bool& found,
                                                uint32_t& pos) {
    uint32_t l, h;
    n2x_inline(P, narrow, C, lo, hi, x, wq, dq1, sub, l, h, pos);
    while (l < h) {
        const uint32_t mid = (l + h) >> 1;
        const uint32_t p = narrow ? static_cast<uint32_t>(__ldg(reinterpret_cast<const unsigned short*>(I) + mid))
                                  : __ldg(I + mid);
        ++probes;
        if (n2x_S(wq, dq1, p, mid, sub) <= x) { l = mid + 1; pos = p; } else h = mid;
    }
    found = l > lo;   // l - 1 is the last true rank, pos = I[l - 1]
    return l - 1;
}

// One thread per walker: the walkers are independent and a step is a short chain of
// dependent sector loads, so thread-level parallelism (up to 2,048 walkers per SM in
// flight) hides the latency that a warp-per-walker kernel exposes.  Per step: the
// record of the entry the walker arrived by (its vertex, row, degree and the step's
// specials), the binary search, and the path store.
#ifndef N2X_MINB
#define N2X_MINB 3   // <= 80 registers, 768 walkers per SM (A/B r02 cfg3: 80 regs 10.1 ms; 64 regs + spills 11.6 ms; 128 regs 11.9 ms)
#endif
__global__ void __launch_bounds__(256, N2X_MINB) k_node2vec_idx(N2xArgs a) {
    const uint32_t wq = a.wq, w1 = a.w1, wp = a.wp;
    const int64_t dq1 = static_cast<int64_t>(wq) - w1, dqp = static_cast<int64_t>(wq) - wp;   // may be negative
    unsigned long long steps = 0, probes_all = 0;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < a.n; w += nthreads) {
        uint32_t* row = a.path + w * (static_cast<uint64_t>(a.L) + 1);
        const uint32_t seed = a.seeds[w];
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        row[0] = seed;
        if (a.L == 0) continue;
        // step 0: uniform over N(seed) (R16)
        const int64_t b0 = __ldg(a.rp + seed);
        const uint32_t d0 = static_cast<uint32_t>(__ldg(a.rp + seed + 1) - b0);
        if (d0 == 0) {   // isolated seed: the walk ends (R20)
            for (int32_t t = 1; t <= a.L; ++t) row[t] = NONE;
            continue;
        }
        uint64_t e = static_cast<uint64_t>(b0) +
                     below(draw_u64(a.key, inst, 0u, 0u, word3(PURPOSE_EDGE, 0, 0)), d0);
        ++steps;
        for (int32_t t = 1;; ++t) {
            const uint4 ra = __ldg(a.rec + N2X_U4 * e), rb = __ldg(a.rec + N2X_U4 * e + 1);
            const void* P = a.rec + N2X_U4 * e + 2;
            row[t] = rb.x;                          // the vertex this entry leads to
            if (t == a.L) break;
            // step t at v = rb.x, arrived from prev by entry e (d >= 1: prev is in N(v))
            const uint64_t U = draw_u64(a.key, inst, static_cast<uint32_t>(t), 0u, word3(PURPOSE_EDGE, 0, 0));
            const uint64_t rs = rb.y | (static_cast<uint64_t>(rb.z & 0xFFu) << 32);
            const uint32_t d = rb.z >> 8;
            const uint32_t C = ra.y >> 8, ppos = ra.z, mb = ra.w;
            const uint32_t* I = a.idx + (ra.x | (static_cast<uint64_t>(ra.y & 0xFFu) << 32));
            const uint64_t T = static_cast<uint64_t>(wq) * (d - C - 1) + static_cast<uint64_t>(w1) * C + wp;
            const int64_t x = static_cast<int64_t>(below(U, T));   // < 2^56
            const int64_t Sp = n2x_S(wq, dq1, ppos, mb, 0);          // S at prev's position
            uint32_t probes = 0, pos = 0, s;
            if (x >= Sp && x < Sp + wp) {
                s = ppos;                                   // prev's own region
            } else {
                // before prev: members [0, mb); after prev: members [mb, C), S one (wq - wp) lower
                const bool after = x >= Sp;
                const int64_t sub = after ? dqp : 0;
                bool found = false;
                const uint32_t j = n2x_last_le(I, P, n2x_narrow(d), C, after ? mb : 0, after ? C : mb, x, wq, dq1, sub,
                                               probes, found, pos);
                if (found) {
                    const int64_t Sm = n2x_S(wq, dq1, pos, j, sub);
                    s = x < Sm + w1 ? pos : pos + 1 + n2x_div(x - Sm - w1, a);
                } else {
                    s = after ? ppos + 1 + n2x_div(x - Sp - wp, a) : n2x_div(x, a);
                }
            }
            probes_all += probes;
            ++steps;
            e = rs + s;
        }
    }
    // sector model (32 B sectors): the edge record (N2X_U4 / 2 sectors) + the probes per step,
    // + 4 B path (step 0: the seed's row_ptr pair instead of a record)
    steps = warp_sum(steps);
    probes_all = warp_sum(probes_all);
    if (lane_id() == 0 && steps) {
        atomicAdd(a.counters + 1, steps);
        atomicAdd(a.counters + 2, probes_all);
        atomicAdd(a.counters + 3, 32ull * ((N2X_U4 / 2) * steps + probes_all) + 4ull * steps);
    }
}

// ---- A step's search state (shared by the kernels below).
struct N2xSearch {          // one walker's step in flight
    uint64_t rs;            // row start of v
    const uint32_t* I;      // member positions of the entry (u16 pairs when narrow)
    int64_t x, Sp, sub;
    uint32_t C, ppos, mb, lo, l, h, pos, s;
    bool after, done, narrow;
};

// record -> the step's search state (prev's own region resolves at once)
__device__ __forceinline__ void n2x_setup(const N2xArgs& a, uint4 ra, uint4 rb, const void* P, uint64_t U,
                                          int64_t dq1, int64_t dqp, N2xSearch& q) {
    const uint32_t wq = a.wq, w1 = a.w1, wp = a.wp;
    q.rs = rb.y | (static_cast<uint64_t>(rb.z & 0xFFu) << 32);
    const uint32_t d = rb.z >> 8;
    q.C = ra.y >> 8; q.ppos = ra.z; q.mb = ra.w;
    q.I = a.idx + (ra.x | (static_cast<uint64_t>(ra.y & 0xFFu) << 32));
    q.narrow = n2x_narrow(rb.z >> 8);
    const uint64_t T = static_cast<uint64_t>(wq) * (d - q.C - 1) + static_cast<uint64_t>(w1) * q.C + wp;
    q.x = static_cast<int64_t>(below(U, T));
    q.Sp = n2x_S(wq, dq1, q.ppos, q.mb, 0);
    q.done = false;
    q.pos = 0;
    if (q.x >= q.Sp && q.x < q.Sp + wp) { q.s = q.ppos; q.done = true; q.l = q.h = 0; return; }
    q.after = q.x >= q.Sp;
    q.sub = q.after ? dqp : 0;
    q.lo = q.after ? q.mb : 0;
    n2x_inline(P, n2x_narrow(d), q.C, q.lo, q.after ? q.C : q.mb, q.x, wq, dq1, q.sub, q.l, q.h, q.pos);
}

// search finished: the pick's position in N(v)
__device__ __forceinline__ uint32_t n2x_finish(const N2xArgs& a, int64_t dq1, const N2xSearch& q) {
    if (q.done) return q.s;
    const uint32_t wq = a.wq, w1 = a.w1, wp = a.wp;
    if (q.l > q.lo) {
        const int64_t Sm = n2x_S(wq, dq1, q.pos, q.l - 1, q.sub);
        return q.x < Sm + w1 ? q.pos : q.pos + 1 + n2x_div(q.x - Sm - w1, a);
    }
    return q.after ? q.ppos + 1 + n2x_div(q.x - q.Sp - wp, a) : n2x_div(q.x, a);
}

// ---- TMA variant: the records (and the probed member positions) are fetched by 1-D bulk
// copies (cp.async.bulk, the Tensor Memory Accelerator) into shared memory and completed on an
// mbarrier per group of 32 walkers.  Measured on this GPU, random 64 B records reach ~2.2 TB/s
// through the TMA against ~0.95 TB/s through vector loads (profiles/r02_random_gather_tma.txt):
// the bulk copies keep more bytes in flight per SM than the load unit's outstanding misses.
// A warp runs N2X_TMA_K groups of 32 walkers round-robin (one group computes while the
// others' copies are in flight; K = 1 measured best: the register budget of one group keeps
// 32 warps per SM); the walkers of a group advance in lock step (same t).  The member-position
// probes stay vector loads through L1 (hub lists are reused across walkers: 45 % L1 hits),
// (A/B r02: member probes by 16 B bulk copies 10.4 ms, a splitter gap fetched whole by one bulk
// copy 9.17 ms, both against 8.16 ms through L1 -- removed).
#ifndef N2X_TMA
#define N2X_TMA 1   // node2vec index walks through the TMA kernel (A/B r02 cfg3: 8.28 ms vs 10.14 ms with vector loads)
#endif
#ifndef N2X_TICKET
#define N2X_TICKET 1   // groups from a global atomic ticket (else a static grid-stride assignment)
#endif
#ifndef N2X_TMA_K
#define N2X_TMA_K 1   // A/B r02 cfg3: K = 1 8.28 ms; K = 2 9.54 ms (80 regs) / 13.6 ms (64 regs + stack)
#endif
#ifndef N2X_TMA_WARPS
#define N2X_TMA_WARPS 4   // 4-warp blocks, 8 per SM (A/B cfg3: 5.94 vs 6.02 ms with 8-warp blocks, 4 per SM)
#endif
#ifndef N2X_SMEM_STRIDE
#define N2X_SMEM_STRIDE (N2X_U4 + 1)   // uint4 per lane slot of the staged records (N2X_U4 = unpadded)
#endif
__device__ __forceinline__ uint32_t n2x_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void n2x_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(n2x_smem(dst)), "l"(src), "r"(bytes), "r"(n2x_smem(bar)) : "memory");
}
__device__ __forceinline__ void n2x_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(n2x_smem(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void n2x_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(n2x_smem(bar)), "r"(parity) : "memory");
}

struct N2xGroup {           // one group of 32 walkers (per-lane fields)
    uint64_t w;             // walker id (>= n: no walker on this lane)
    uint64_t e;             // the entry the walker arrived by
    N2xSearch q;            // the step in flight
    int32_t t;              // step (group-uniform)
    uint32_t parity;        // mbarrier phase
    bool live;              // group-uniform: the group holds walkers
};

#ifndef N2X_TMA_MINB
#define N2X_TMA_MINB 8   // x 4 warps, <= 64 registers: 32 warps / SM (A/B r02 cfg3: 95 regs 11.45 ms, 64 regs 8.28, 48 regs + stack 9.14)
#endif
__global__ void __launch_bounds__(N2X_TMA_WARPS * 32, N2X_TMA_MINB) k_node2vec_tma(N2xArgs a) {
    constexpr int K = N2X_TMA_K;
    // one record per lane at a stride of an odd number of uint4: a warp's uint4 reads of the
    // records then hit 8 distinct 16 B bank groups per 8-lane phase (conflict-free) -- 64 B
    // records at a 64 B stride were a 4-way conflict per phase (ncu r02: 75 % excessive wavefronts)
    __shared__ __align__(128) uint4 recs[N2X_TMA_WARPS][K][32][N2X_SMEM_STRIDE];
    __shared__ __align__(8) uint64_t bars[N2X_TMA_WARPS][K];
    const int lane = lane_id(), wib = threadIdx.x >> 5;
    const uint32_t wq = a.wq, w1 = a.w1, wp = a.wp;
    const int64_t dq1 = static_cast<int64_t>(wq) - w1, dqp = static_cast<int64_t>(wq) - wp;
    unsigned long long steps = 0, probes_all = 0;
    if (lane == 0)
        for (int k = 0; k < K; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(n2x_smem(&bars[wib][k])));
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#if !N2X_TICKET
    const uint64_t gstride = static_cast<uint64_t>(gridDim.x) * N2X_TMA_WARPS * K;   // groups in flight grid-wide
    uint64_t next_group = (static_cast<uint64_t>(blockIdx.x) * N2X_TMA_WARPS + wib) * K;
#endif
    N2xGroup G[K] = {};

    auto issue_records = [&](int k) {
        const bool me = G[k].w < a.n;
        const uint32_t cnt = __popc(__ballot_sync(FULL, me));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // our reads of the slot before the copy
        if (lane == 0) n2x_expect(&bars[wib][k], cnt * (16u * N2X_U4));
        __syncwarp();
        if (me) n2x_bulk(&recs[wib][k][lane][0], a.rec + N2X_U4 * G[k].e, 16u * N2X_U4, &bars[wib][k]);
    };
    // a new group: step 0 (uniform, R16) for each lane's walker, then its first record
    auto start_group = [&](int k) {
        for (;;) {
#if N2X_TICKET
            // the next group from a global ticket (a9: warps fetch work dynamically, so warps whose
            // walkers sat on hubs do not leave the others waiting at the end)
            unsigned long long tk = 0;
            if (lane == 0) tk = atomicAdd(a.counters + 7, 1ull);
            const uint64_t gi = __shfl_sync(FULL, tk, 0);
#else
            const uint64_t gi = next_group;
            next_group += (gi % K == static_cast<uint64_t>(K - 1)) ? gstride - (K - 1) : 1;
#endif
            const uint64_t w = gi * 32 + lane;
            G[k].live = gi * 32 < a.n;
            if (!G[k].live) return;
            G[k].w = w < a.n ? w : ~0ull;
            G[k].t = 1;
            if (G[k].w != ~0ull) {
                uint32_t* row = a.path + w * (static_cast<uint64_t>(a.L) + 1);
                const uint32_t seed = a.seeds[w];
                row[0] = seed;
                const int64_t b0 = __ldg(a.rp + seed);
                const uint32_t d0 = static_cast<uint32_t>(__ldg(a.rp + seed + 1) - b0);
                if (a.L == 0) {
                    G[k].w = ~0ull;
                } else if (d0 == 0) {   // isolated seed: the walk ends (R20)
                    for (int32_t t = 1; t <= a.L; ++t) row[t] = NONE;
                    G[k].w = ~0ull;
                } else {
                    G[k].e = static_cast<uint64_t>(b0) +
                             below(draw_u64(a.key, a.base + static_cast<uint32_t>(w), 0u, 0u, word3(PURPOSE_EDGE, 0, 0)), d0);
                    ++steps;
                }
            }
            if (__ballot_sync(FULL, G[k].w < a.n)) { issue_records(k); return; }
            // nothing to fetch in this group (all isolated / L = 0): take the next one
        }
    };
    for (int k = 0; k < K; ++k) { G[k].parity = 0; G[k].live = false; }
    for (int k = 0; k < K; ++k) start_group(k);
    for (;;) {
        bool any = false;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (!G[k].live) continue;
            any = true;
            n2x_wait(&bars[wib][k], G[k].parity);
            G[k].parity ^= 1u;
            const bool me = G[k].w < a.n;
            {   // records arrived: path entry, then the step's search
                if (me) {
                    const uint4 ra = recs[wib][k][lane][0], rb = recs[wib][k][lane][1];
                    const void* P = &recs[wib][k][lane][2];
                    uint32_t* row = a.path + G[k].w * (static_cast<uint64_t>(a.L) + 1);
                    row[G[k].t] = rb.x;
                    if (G[k].t < a.L) {
                        const uint64_t U = draw_u64(a.key, a.base + static_cast<uint32_t>(G[k].w),
                                                    static_cast<uint32_t>(G[k].t), 0u, word3(PURPOSE_EDGE, 0, 0));
                        n2x_setup(a, ra, rb, P, U, dq1, dqp, G[k].q);
                    }
                }
                if (G[k].t == a.L) {   // the group's walks are complete
                    start_group(k);
                    continue;
                }
            }
            __syncwarp();
            if (me) {   // the member positions through L1 (hub lists are reused across walkers; whole
                        // 128 B lines from DRAM: .L2::64B measured 7.81 vs 7.54 ms on cfg3)
                while (G[k].q.l < G[k].q.h) {
                    const uint32_t mid = (G[k].q.l + G[k].q.h) >> 1;
                    CSAW_DASSERT(static_cast<uint64_t>(G[k].q.I - a.idx) + (G[k].q.narrow ? mid / 2 : mid) < a.idx_n);
                    const uint32_t p = G[k].q.narrow
                                           ? static_cast<uint32_t>(__ldg(reinterpret_cast<const unsigned short*>(G[k].q.I) + mid))
                                           : __ldg(G[k].q.I + mid);
                    ++probes_all;
                    if (n2x_S(wq, dq1, p, mid, G[k].q.sub) <= G[k].q.x) { G[k].q.l = mid + 1; G[k].q.pos = p; }
                    else G[k].q.h = mid;
                }
            }
            // every lane's region is known: finish the step, fetch the next records
            if (me) {
                G[k].e = G[k].q.rs + n2x_finish(a, dq1, G[k].q);
                ++steps;
            }
            ++G[k].t;
            issue_records(k);
        }
        if (!any) break;
    }
    steps = warp_sum(steps);
    probes_all = warp_sum(probes_all);
    if (lane == 0 && steps) {
        atomicAdd(a.counters + 1, steps);
        atomicAdd(a.counters + 2, probes_all);
        atomicAdd(a.counters + 3, 32ull * ((N2X_U4 / 2) * steps + probes_all) + 4ull * steps);
    }
}


csaw_status launch_node2vec_index(const csaw_graph* g, const uint32_t* seeds, uint64_t n, int32_t L, uint32_t base,
                                  uint2 key, uint32_t* path, unsigned long long* counters, uint32_t wp, uint32_t w1,
                                  uint32_t wq, cudaStream_t st) {
    int32_t sh = -1;
    for (int b = 0; b < 31; ++b)
        if (wq == (1u << b)) sh = b;
    N2xArgs a{g->row_ptr, g->n2x_rec, g->n2x_idx, g->n2x_total + 8, seeds, n, L, base, key, path, counters, wp, w1, wq, sh,
              1.0 / static_cast<double>(wq)};
    const uint64_t resident = static_cast<uint64_t>(g->num_sms) * 2048;
    if (N2X_TMA) {
        // persistent: as many blocks as are resident at once (each warp then loops over groups)
        static int per_sm = 0;
        if (per_sm == 0 &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_node2vec_tma, N2X_TMA_WARPS * 32, 0) != cudaSuccess) {
            cudaGetLastError();
            per_sm = 1;
        }
        const uint64_t groups = (n + 31) / 32;
        const uint64_t per_block = N2X_TMA_WARPS * N2X_TMA_K;
        const uint64_t blocks = std::min<uint64_t>((groups + per_block - 1) / per_block,
                                                   static_cast<uint64_t>(g->num_sms) * std::max(per_sm, 1));
        k_node2vec_tma<<<static_cast<int>(std::max<uint64_t>(1, blocks)), N2X_TMA_WARPS * 32, 0, st>>>(a);
    } else {
        const uint64_t threads = std::min<uint64_t>(n, resident);
        const int grid = static_cast<int>(std::max<uint64_t>(1, (threads + 255) / 256));
        k_node2vec_idx<<<grid, 256, 0, st>>>(a);
    }
    note_launch();
    CSAW_CUDA(cudaGetLastError());
    return CSAW_OK;
}

}  // namespace csaw
