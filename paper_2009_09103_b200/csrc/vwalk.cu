// vwalk.cu — walks whose EdgeBias is a per-edge stream (vscan.cuh): the edge-weight walk
// (CSAW_BIAS_WEIGHT, EdgeBias = w(e), Eq. 3, float path R28) and the degree-biased
// walk over the materialised bias deg(col[e]) (CSAW_GRAPH_EDGE_BIAS; biased DeepWalk P:172).
//
// Every step is the paper's Select (§4.1): evaluate the pool's biases, build the CTPS by a
// warp scan, one keyed Philox draw, inverse transform search
// -- nothing is cached across steps.  A group of G warps walks one walker and
// splits each pool's chunks between them (the hub route of SURVEY D7: few walkers with
// large pools still fill the GPU); G = 1 when walkers alone fill it.  The chunking, hence
// every sum, depends only on the pool, so G never changes a result (R7).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "vscan.cuh"

namespace csaw {

constexpr int VW_WARPS = 8;   // warps per block

struct VWalkArgs {
    const int64_t* __restrict__ rp;
    const uint32_t* __restrict__ col;
    const uint32_t* __restrict__ seeds;
    uint64_t n;
    int32_t L;
    uint32_t base;
    uint2 key;
    uint32_t* __restrict__ path;
    unsigned long long* __restrict__ counters;   // [0] neighbours scanned, [1] steps
};

template <int G>
__device__ __forceinline__ void group_bar(int grp) {
    if constexpr (G > 1) asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(G * 32) : "memory");
    else __syncwarp();
}

template <class E, int G>
__global__ void __launch_bounds__(VW_WARPS * 32, 4) k_walk_vscan(VWalkArgs a, const E* __restrict__ eb) {
    using Acc = typename VTraits<E>::Acc;
    constexpr int NG = VW_WARPS / G;   // walker groups per block
    __shared__ Acc tab_all[NG][TAB];
    __shared__ VGroupShared<E> sh_all[NG];
    const int warp = threadIdx.x >> 5, grp = warp / G, gw = warp % G;
    const int lane = lane_id();
    Acc* tab = tab_all[grp];
    VGroupShared<E>* sh = &sh_all[grp];
    auto bar = [grp]() { group_bar<G>(grp); };
    unsigned long long scanned = 0, steps = 0;
    for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * NG + grp; w < a.n; w += static_cast<uint64_t>(gridDim.x) * NG) {
        uint32_t cur = a.seeds[w];
        const uint32_t inst = a.base + static_cast<uint32_t>(w);
        uint32_t* row = a.path + w * (static_cast<uint64_t>(a.L) + 1);
        uint32_t buf = NONE;   // path entries buffered one per lane, flushed as 128 B stores (warp 0)
        if (lane == 0) buf = cur;
        for (int32_t t = 0; t < a.L; ++t) {
            uint32_t nxt = NONE;
            if (cur != NONE) {
                const int64_t b0 = __ldg(a.rp + cur);
                const uint32_t d = static_cast<uint32_t>(__ldg(a.rp + cur + 1) - b0);
                if (d > 0) {
                    VPool<E> P;
                    P.init(eb, a.col, static_cast<uint64_t>(b0), d);
                    const VCtps<E> C = vscan_build<E, G, false>(P, tab, sh, gw, bar);
                    if (gw == 0) {
                        const uint64_t U = draw_u64(a.key, inst, static_cast<uint32_t>(t), 0u, word3(PURPOSE_EDGE, 0, 0));
                        nxt = vscan_select_wr(P, C, tab, U);
                        scanned += d;
                        ++steps;
                    }
                    if constexpr (G > 1) {
                        if (gw == 0 && lane == 0) sh->word = nxt;
                        bar();
                        nxt = sh->word;
                    }
                }
            }
            cur = nxt;
            if (gw == 0) {
                const int32_t pi = t + 1;
                if ((pi & 31) == lane) buf = cur;
                if ((pi & 31) == 31 || pi == a.L) {
                    const int32_t idx = (pi & ~31) + lane;
                    if (idx <= pi) row[idx] = buf;
                }
            }
        }
        if (a.L == 0 && gw == 0 && lane == 0) row[0] = buf;
        if constexpr (G > 1) bar();   // the next walker's first build reuses tab / sh
    }
    if (lane == 0 && gw == 0) {
        if (scanned) atomicAdd(a.counters + 0, scanned);
        if (steps) atomicAdd(a.counters + 1, steps);
    }
}

// G: warps per walker -- the widest group with every walker resident at once (32 warps per
// SM at 64 registers); few walkers with large pools then still fill the GPU (results
// identical, R7).
static int vwalk_group(const csaw_graph* g, int64_t n) {
    const int64_t resident = static_cast<int64_t>(g->num_sms) * 32;
    int G = 1;
    while (G < 8 && n * (2 * G) <= resident) G *= 2;
    return G;
}

template <class E>
static void launch_vwalk(const csaw_graph* g, const VWalkArgs& a, const E* eb, int G, cudaStream_t st) {
    const int64_t groups_per_block = VW_WARPS / G;
    const int64_t resident_groups = static_cast<int64_t>(g->num_sms) * (64 / G);
    const int64_t groups = std::min<int64_t>(static_cast<int64_t>(a.n), resident_groups);
    const int grid = static_cast<int>(std::max<int64_t>(1, (groups + groups_per_block - 1) / groups_per_block));
    switch (G) {
        case 1: k_walk_vscan<E, 1><<<grid, VW_WARPS * 32, 0, st>>>(a, eb); break;
        case 2: k_walk_vscan<E, 2><<<grid, VW_WARPS * 32, 0, st>>>(a, eb); break;
        case 4: k_walk_vscan<E, 4><<<grid, VW_WARPS * 32, 0, st>>>(a, eb); break;
        default: k_walk_vscan<E, 8><<<grid, VW_WARPS * 32, 0, st>>>(a, eb); break;
    }
}

csaw_status launch_walk_vscan(const csaw_graph* g, bool weights, const uint32_t* seeds, uint64_t n, int32_t L,
                              uint32_t base, uint2 key, uint32_t* path, unsigned long long* counters, int group,
                              cudaStream_t st) {
    VWalkArgs a{g->row_ptr, g->col, seeds, n, L, base, key, path, counters};
    const int G = group > 0 ? group : vwalk_group(g, static_cast<int64_t>(n));
    if (weights) launch_vwalk<float>(g, a, g->w, G, st);
    else launch_vwalk<uint32_t>(g, a, g->ebias, G, st);
    note_launch();
    CSAW_CUDA(cudaGetLastError());
    return CSAW_OK;
}

}  // namespace csaw
