// capi.cu — C ABI entry points, graph creation / validation, error plumbing.
//
// csaw_graph_create copies and validates a CSR on the device (the paper's L0
// graph storage, §5.1 P:808-813 / Table 2 "Size (of CSR)") and precomputes the
// degree array used by every degree bias (one 4-byte gather per neighbour
// instead of two row_ptr reads).
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "internal.h"
#include "select.cuh"
#include "wix.cuh"
#include "util.cuh"

namespace csaw {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }

csaw_status cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                  cudaGetErrorString(e), what, file, line);
    set_error(buf);
    if (e == cudaErrorMemoryAllocation) return CSAW_ERR_NO_MEMORY;
    return CSAW_ERR_CUDA;
}

Scratch::~Scratch() { release_all(); }

void Scratch::release_all() {
    for (auto& b : bufs_)
        if (b.p) cudaFree(b.p);
    bufs_.clear();
}

csaw_status Scratch::get(int slot, size_t bytes, void** out) {
    if (slot < 0) return fail(CSAW_ERR_INVALID_ARG, "bad scratch slot");
    if (static_cast<size_t>(slot) >= bufs_.size()) bufs_.resize(slot + 1);
    Buf& b = bufs_[slot];
    if (bytes == 0) bytes = 16;
    if (b.n < bytes) {
        if (b.p) {
            CSAW_CUDA(cudaDeviceSynchronize());   // buffer may still be in use by queued work
            CSAW_CUDA(cudaFree(b.p));
            b.p = nullptr;
            b.n = 0;
        }
        const size_t want = std::max(bytes, b.n + b.n / 2);
        cudaError_t e = cudaMalloc(&b.p, want);
        if (e != cudaSuccess) {
            e = cudaMalloc(&b.p, bytes);
            if (e != cudaSuccess) { b.p = nullptr; return cuda_fail(e, "cudaMalloc(scratch)", __FILE__, __LINE__); }
            b.n = bytes;
        } else {
            b.n = want;
        }
    }
    *out = b.p;
    return CSAW_OK;
}

size_t Scratch::bytes_held() const {
    size_t s = 0;
    for (auto& b : bufs_) s += b.n;
    return s;
}

PinnedBuf::~PinnedBuf() {
    if (p_) cudaFreeHost(p_);
}

csaw_status PinnedBuf::get(size_t bytes, void** out) {
    if (n_ < bytes) {
        if (p_) cudaFreeHost(p_);
        p_ = nullptr;
        n_ = 0;
        CSAW_CUDA(cudaMallocHost(&p_, bytes));
        n_ = bytes;
    }
    *out = p_;
    return CSAW_OK;
}

PtrKind ptr_kind(const void* p, int device) {
    if (!p) return PtrKind::Pageable;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return PtrKind::Pageable;
    }
    if (a.type == cudaMemoryTypeDevice) return a.device == device ? PtrKind::Device : PtrKind::OtherDevice;
    if (a.type == cudaMemoryTypeManaged) return PtrKind::Device;
    if (a.type == cudaMemoryTypeHost) return PtrKind::Pinned;
    return PtrKind::Pageable;
}

bool is_device_ptr(const void* p, int device) { return ptr_kind(p, device) == PtrKind::Device; }

CallOrder::CallOrder(const csaw_graph* g_, cudaStream_t st_) : g(g_), st(st_) {
    if (g && g->ev_done) cudaStreamWaitEvent(st, g->ev_done, 0);
}

CallOrder::~CallOrder() {
    if (g && g->ev_done) cudaEventRecord(g->ev_done, st);
}

// Device-side address of pinned (page-locked) host memory, or nullptr for pageable memory.
void* pinned_device_ptr(void* p) {
    if (!p) return nullptr;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

csaw_status begin_call(const csaw_graph* g) {
    clear_error();
    if (!g) return fail(CSAW_ERR_INVALID_ARG, "graph is NULL");
    CSAW_CUDA(cudaSetDevice(g->device));
    return CSAW_OK;
}

thread_local uint64_t tl_launches = 0;

csaw_status stats_begin(const csaw_graph* g, cudaStream_t st) {
    g->stats = csaw_run_stats{};
    g->hot_used = 0;
    g->pending_counters = nullptr;
    tl_launches = 0;
    CSAW_CUDA(cudaEventRecord(g->ev0, st));
    return CSAW_OK;
}

csaw_status hot_begin(const csaw_graph* g, cudaStream_t st) {
    const size_t need = static_cast<size_t>(g->hot_used) * 2 + 2;
    while (g->hot_ev.size() < need) {
        cudaEvent_t e;
        CSAW_CUDA(cudaEventCreate(&e));
        g->hot_ev.push_back(e);
    }
    CSAW_CUDA(cudaEventRecord(g->hot_ev[g->hot_used * 2], st));
    return CSAW_OK;
}

csaw_status hot_end(const csaw_graph* g, cudaStream_t st) {
    CSAW_CUDA(cudaEventRecord(g->hot_ev[g->hot_used * 2 + 1], st));
    ++g->hot_used;
    return CSAW_OK;
}

csaw_status stats_end(const csaw_graph* g, cudaStream_t st) {
    g->stats.kernel_launches = tl_launches;
    g->stats.hot_launches = static_cast<uint64_t>(g->hot_used);
    CSAW_CUDA(cudaEventRecord(g->ev1, st));
    return CSAW_OK;
}

// ---------------------------------------------------------------- validation kernels
struct ValidateOut {
    unsigned long long bad_rowptr;     // first v with row_ptr[v+1] < row_ptr[v] (+1), 0 = ok
    unsigned long long bad_col;        // first e with col[e] >= V (+1)
    unsigned long long unsorted;       // count of rows not strictly ascending
    unsigned long long max_deg;
    unsigned long long nonisolated;
    unsigned long long bad_weight;     // first e with weights[e] < 0 or not finite (+1)
};

__global__ void k_validate_weights(const float* __restrict__ w, int64_t E, ValidateOut* out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
        if (!(w[e] >= 0.0f && isfinite(w[e]))) atomicMin(&out->bad_weight, static_cast<unsigned long long>(e + 1));
}

// materialised degree bias per CSR entry (vscan.cuh): ebias[e] = deg(col[e])
__global__ void k_build_ebias(const uint32_t* __restrict__ col, const uint32_t* __restrict__ deg, int64_t E,
                              uint32_t* __restrict__ ebias) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
        ebias[e] = __ldg(deg + __ldg(col + e));
}

__global__ void k_validate_rows(const int64_t* __restrict__ rp, int64_t V, uint32_t* __restrict__ deg,
                                ValidateOut* out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = rp[v], b = rp[v + 1];
        if (b < a) atomicMin(&out->bad_rowptr, static_cast<unsigned long long>(v + 1));
        const int64_t d = b - a;
        deg[v] = d > 0 ? static_cast<uint32_t>(d) : 0u;
        if (d > 0) {
            atomicMax(&out->max_deg, static_cast<unsigned long long>(d));
            atomicAdd(&out->nonisolated, 1ull);
        }
    }
}

__global__ void k_validate_cols(const uint32_t* __restrict__ col, int64_t E, int64_t e0, int64_t V, ValidateOut* out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
        if (static_cast<int64_t>(col[e]) >= V) atomicMin(&out->bad_col, static_cast<unsigned long long>(e0 + e + 1));
}

// warp per row: strictly ascending check
__global__ void k_validate_sorted(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col, int64_t v0,
                                  int64_t v1, ValidateOut* out) {
    const int lane = lane_id();
    for (uint64_t v = v0 + global_warp_id(); v < static_cast<uint64_t>(v1); v += total_warps()) {
        const int64_t a = rp[v], b = rp[v + 1];
        bool bad = false;
        for (int64_t e = a + lane; e + 1 < b; e += 32) bad |= col[e] >= col[e + 1];
        if (__any_sync(FULL, bad) && lane == 0) atomicAdd(&out->unsorted, 1ull);
    }
}

// Static-bias CTPS cache ("caching transition probability", R25): warp per
// row, the same Kogge-Stone u64 scan the select kernels run per step.
__global__ void k_build_cps(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                            const uint32_t* __restrict__ deg, int64_t V, uint64_t* __restrict__ cps,
                            uint32_t* __restrict__ npos) {
    const int lane = lane_id();
    for (uint64_t v = global_warp_id(); v < static_cast<uint64_t>(V); v += total_warps()) {
        const int64_t a = rp[v], b = rp[v + 1];
        uint64_t carry = 0;
        uint32_t pos = 0;
        for (int64_t e0 = a; e0 < b; e0 += 32) {
            const int64_t e = e0 + lane;
            const uint32_t bias = e < b ? __ldg(deg + __ldg(col + e)) : 0u;
            const uint64_t incl = warp_incl_scan(static_cast<uint64_t>(bias)) + carry;
            if (e < b) cps[e] = incl;
            carry = __shfl_sync(FULL, incl, 31);
            pos += __popc(__ballot_sync(FULL, bias > 0));
        }
        if (lane == 0) npos[v] = pos;
    }
}

// B-tree index over the cached prefix (select.cuh CpsTree): sizes, then levels.
__device__ __forceinline__ uint64_t bt_size_of(uint64_t d) {
    uint64_t s = 0, nk = d;
    while (nk > 32) { nk = (nk + 31) / 32; s += nk; }
    return s;
}

struct BtSize {
    const int64_t* rp;
    __device__ __forceinline__ uint64_t operator()(uint64_t v) const { return bt_size_of(rp[v + 1] - rp[v]); }
};

// nmp[e] = row_ptr[u] << 24 | deg(u) for u = col[e]: a walk step that picks entry e
// learns the next vertex's row and degree in the same round (no row_ptr lookup).
__global__ void k_build_nmp(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col, int64_t E,
                            uint64_t* __restrict__ nmp) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t u = col[e];
        const int64_t a = rp[u];
        nmp[e] = (static_cast<uint64_t>(a) << 24) | static_cast<uint64_t>(rp[u + 1] - a);
    }
}

// nrec[e] = {u, deg(u), row_ptr[u] lo, hi} for u = col[e]: the entry an MDRW step picks and
// the new pool vertex's row and degree in one 16 B read (one random DRAM access, not two).
__global__ void k_build_nrec(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col, int64_t E,
                             uint4* __restrict__ nrec) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t u = col[e];
        const int64_t a = rp[u];
        nrec[e] = make_uint4(u, static_cast<uint32_t>(rp[u + 1] - a), static_cast<uint32_t>(a),
                             static_cast<uint32_t>(static_cast<uint64_t>(a) >> 32));
    }
}

__global__ void k_build_bt(const int64_t* __restrict__ rp, const uint64_t* __restrict__ cps,
                           const uint64_t* __restrict__ bt_off, int64_t V, uint64_t* __restrict__ bt) {
    const int lane = lane_id();
    for (uint64_t v = global_warp_id(); v < static_cast<uint64_t>(V); v += total_warps()) {
        const int64_t beg = rp[v];
        const uint64_t d = static_cast<uint64_t>(rp[v + 1] - beg);
        if (d <= 32) continue;
        uint64_t n[8];
        int K = 0;
        n[0] = d;
        while (n[K] > 32 && K < 7) { n[K + 1] = (n[K] + 31) / 32; ++K; }
        uint64_t off[8];
        uint64_t acc = 0;
        for (int k = K; k >= 1; --k) { off[k] = acc; acc += n[k]; }
        const uint64_t base = bt_off[v];
        for (int k = 1; k <= K; ++k) {
            for (uint64_t j = lane; j < n[k]; j += 32) {
                const uint64_t src = min(j * 32 + 31, n[k - 1] - 1);
                bt[base + off[k] + j] = (k == 1) ? cps[beg + src] : bt[base + off[k - 1] + src];
            }
            __syncwarp();
        }
    }
}


// ---------------------------------------------------------------- narrow walk index (wix.cuh)
// Every row total T = cps[row end - 1] must be < 2^32 for the u32 index.
__global__ void k_wix_check(const int64_t* __restrict__ rp, const uint64_t* __restrict__ cps, int64_t V,
                            unsigned int* __restrict__ wide) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = rp[v + 1];
        if (b > rp[v] && cps[b - 1] >> 32) atomicOr(wide, 1u);
    }
}

template <int FL>
struct WixSize {
    const int64_t* rp;
    __device__ __forceinline__ uint64_t operator()(uint64_t v) const {
        return WixShape<FL>::index_size(static_cast<uint32_t>(rp[v + 1] - rp[v]));
    }
};

// Warp per row: padded leaf copies, the record, then the internal levels bottom-up
// (level k reads k-1).
template <int FL>
__global__ void k_wix_build(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                            const uint64_t* __restrict__ cps, const uint64_t* __restrict__ woff, int64_t V,
                            uint4* __restrict__ rec, uint32_t* __restrict__ c32p, uint32_t* __restrict__ colp,
                            uint32_t* __restrict__ inn) {
    using W = WixShape<FL>;
    const int lane = lane_id();
    for (uint64_t v = global_warp_id(); v < static_cast<uint64_t>(V); v += total_warps()) {
        const int64_t rb = rp[v];
        const uint32_t d = static_cast<uint32_t>(rp[v + 1] - rb);
        const uint64_t p = W::leaf_pos(static_cast<uint64_t>(rb), v);
        const uint64_t io = woff[v];
        if (lane == 0)   // T = S_d (the caller checked T < 2^32, p < 2^32, io < 2^32)
            rec[v] = make_uint4(static_cast<uint32_t>(p), d, static_cast<uint32_t>(io),
                                d ? static_cast<uint32_t>(cps[rb + d - 1]) : 0u);
        for (uint32_t i = lane; i < d; i += 32) {
            c32p[p + i] = static_cast<uint32_t>(cps[rb + i]);
            colp[p + i] = col[rb + i];
        }
        __syncwarp();
        const int K = W::levels(d);
        uint64_t offk[8];
        uint64_t acc = 0;
        for (int k = K; k >= 1; --k) { offk[k] = acc; acc += W::round4(W::count(d, k)); }
        for (int k = 1; k <= K; ++k) {
            const uint32_t nk = W::count(d, k);
            const uint32_t nchild = k == 1 ? d : W::count(d, k - 1);
            const uint32_t span = k == 1 ? FL : WIX_NODE;
            for (uint32_t j = lane; j < nk; j += 32) {
                const uint32_t last = min((j + 1) * span, nchild) - 1;
                inn[io + offk[k] + j] = k == 1 ? c32p[p + last] : inn[io + offk[k - 1] + last];
            }
            __syncwarp();
        }
    }
}

// Vertex heads (wix.cuh): warp per vertex, from the record, the top level and the leaves.
template <int FL>
__global__ void k_head_build(const uint4* __restrict__ rec, const uint32_t* __restrict__ c32p,
                             const uint32_t* __restrict__ colp, const uint32_t* __restrict__ inn, int64_t V,
                             uint32_t* __restrict__ head) {
    using W = WixShape<FL>;
    const int lane = lane_id();
    for (uint64_t v = global_warp_id(); v < static_cast<uint64_t>(V); v += total_warps()) {
        const uint4 r = rec[v];   // {p, d, io, T}
        uint32_t* h = head + v * WIX_HEAD_WORDS;
        const uint32_t d = r.y;
        const int K = W::levels(d);
        for (uint32_t w = lane; w < WIX_HEAD_WORDS; w += 32) {
            uint32_t val = 0;
            if (w == 0) val = d;
            else if (w == 1) val = r.w;
            else if (w == 2) val = r.x;
            else if (w == 3) val = r.z;
            else if (K == 0 && d <= WIX_HEAD_LEAF) {
                const uint32_t i = w - 4;
                if (i < WIX_HEAD_LEAF) val = i < d ? c32p[r.x + i] : 0u;
                else if (i - WIX_HEAD_LEAF < d) val = colp[r.x + (i - WIX_HEAD_LEAF)];
            } else if (K > 0) {
                const uint32_t nK = W::count(d, K);
                if (nK <= WIX_HEAD_TOP && w - 4 < nK) val = inn[r.z + (w - 4)];
            }
            h[w] = val;
        }
    }
}

template <int FL>
static csaw_status build_wix_t(csaw_graph* g, int blocks) {
    using W = WixShape<FL>;
    const int64_t V = g->V, E = g->E;
    uint64_t* woff = nullptr;
    uint64_t* part = nullptr;
    if (cudaMalloc(&woff, sizeof(uint64_t) * (V + 1)) != cudaSuccess ||
        cudaMalloc(&part, sizeof(uint64_t) * (SCAN_MAX_GRID + 8)) != cudaSuccess) {   // accelerator: skip it
        cudaGetLastError();
        if (woff) cudaFree(woff);
        return CSAW_OK;
    }
    csaw_status s = device_scan(WixSize<FL>{g->row_ptr}, static_cast<uint64_t>(V), ScanToArray{woff}, part, nullptr);
    uint64_t total = 0;
    if (s == CSAW_OK && cudaMemcpy(&total, woff + V, sizeof(uint64_t), cudaMemcpyDeviceToHost) != cudaSuccess)
        s = fail(CSAW_ERR_CUDA, "walk index size");
    cudaFree(part);
    const uint64_t nl = W::leaf_total(static_cast<uint64_t>(E), static_cast<uint64_t>(V));
    // u32 record fields: else keep the u64 index
    if (s == CSAW_OK && total + 16 < (uint64_t(1) << 32) && nl < (uint64_t(1) << 32)) {
        if (cudaMalloc(&g->c32, sizeof(uint32_t) * nl) != cudaSuccess ||
            cudaMalloc(&g->wcol, sizeof(uint32_t) * nl) != cudaSuccess ||
            cudaMalloc(&g->winn, sizeof(uint32_t) * (total + 16) + sizeof(uint4) * std::max<int64_t>(V, 1)) != cudaSuccess) {
            // the walk index is an accelerator: without memory for it, walks use the u64 index
            cudaGetLastError();
            if (g->c32) cudaFree(g->c32);
            if (g->wcol) cudaFree(g->wcol);
            if (g->winn) cudaFree(g->winn);
            g->c32 = g->wcol = g->winn = nullptr;
        } else {
            cudaMemset(g->c32, 0, sizeof(uint32_t) * nl);   // padding entries (read, then masked)
            cudaMemset(g->wcol, 0, sizeof(uint32_t) * nl);
            cudaMemset(g->winn, 0, sizeof(uint32_t) * (total + 16));
            // records right after the nodes (total + 16 is a multiple of 4: 16 B aligned)
            g->wrec = reinterpret_cast<uint4*>(g->winn + total + 16);
            k_wix_build<FL><<<blocks, 256>>>(g->row_ptr, g->col, g->cps, woff, V, g->wrec, g->c32, g->wcol, g->winn);
            if (!(g->flags & CSAW_GRAPH_WALK_NO_HEADS) &&
                cudaMalloc(&g->whead, sizeof(uint32_t) * WIX_HEAD_WORDS * std::max<int64_t>(V, 1)) == cudaSuccess)
                k_head_build<FL><<<blocks, 256>>>(g->wrec, g->c32, g->wcol, g->winn, V, g->whead);
            else
                cudaGetLastError();   // heads are an accelerator: walks fall back to the records
            g->winn_entries = total + 16;
            g->wleaf_entries = nl;
        }
    }
    cudaFree(woff);
    return s;
}

// Builds the index unless some row total is >= 2^32 (then walks keep the u64 CpsTree path).
// Leaf fanout 128, or 64 / 32 with CSAW_GRAPH_WALK_LEAF_64 / _32 (cfg2 with vertex heads:
// 128: 2.374, 64: 2.397, 32: 2.522 ms).
static csaw_status build_wix(csaw_graph* g, int blocks) {
    const int leaf = (g->flags & CSAW_GRAPH_WALK_LEAF_32) ? 32 : (g->flags & CSAW_GRAPH_WALK_LEAF_64) ? 64 : 128;
    unsigned int* wide = nullptr;
    CSAW_CUDA(cudaMalloc(&wide, sizeof(unsigned int)));
    CSAW_CUDA(cudaMemset(wide, 0, sizeof(unsigned int)));
    if (g->V > 0) k_wix_check<<<blocks, 256>>>(g->row_ptr, g->cps, g->V, wide);
    unsigned int hw = 0;
    CSAW_CUDA(cudaMemcpy(&hw, wide, sizeof(hw), cudaMemcpyDeviceToHost));
    cudaFree(wide);
    if (hw || g->E <= 0) return CSAW_OK;
    csaw_status s = leaf == 32 ? build_wix_t<32>(g, blocks) : leaf == 64 ? build_wix_t<64>(g, blocks)
                                                               : build_wix_t<128>(g, blocks);
    if (s == CSAW_OK && g->c32) {
        g->wix_leaf = leaf;
        // lanes per walker: 32 (one warp per walker, default) | 16 | 8 (CSAW_GRAPH_WALK_GROUP_*;
        // the sub-warp kernels are slower at cfg2, 3.7 / 4.4 ms vs 2.8 ms: a warp's walkers
        // then wait for the slowest of their dependent-load chains every step)
        const int grp = (g->flags & CSAW_GRAPH_WALK_GROUP_8) ? 8 : (g->flags & CSAW_GRAPH_WALK_GROUP_16) ? 16 : 32;
        g->wix_group = (grp == 16 && leaf >= 64) ? 16 : grp == 8 ? 8 : 32;
    }
    return s;
}

// ---------------------------------------------------------------- bucketed walk index
// CSAW_GRAPH_WALK_BUCKETS (csaw.h): row v's CTPS [0, T) in buckets of width 2^k, k = floor(log2(T / d)),
// each bucket one 128 B line of 8 entries {S_i, u | k_u << 27, first bucket of u, T_u} for the regions
// meeting it; a 9th region turns entry 7 into {S_i, GB_LINK, CSR entry of region i lo, hi}.
constexpr uint32_t GB_EMPTY = 0xFFFFFFFFu;   // S of an unused entry (> every draw: T < 2^32 - 2)
constexpr uint32_t GB_LINK = 0xFFFFFFFFu;    // u field of a link entry (V < 2^27 - 1, so never u | k << 27)
__host__ __device__ __forceinline__ uint32_t gb_shift(uint64_t T, uint64_t d) {
    uint64_t r = T / d;   // mean region width (>= 1 unless some regions are empty)
    uint32_t k = 0;
    while (r > 1) { r >>= 1; ++k; }
    return k;
}
struct GbSize {
    const int64_t* rp;
    const uint64_t* cps;
    __device__ __forceinline__ uint64_t operator()(uint64_t v) const {
        const int64_t b = rp[v], e = rp[v + 1];
        if (e == b) return 0;
        const uint64_t T = cps[e - 1];
        if (T == 0) return 0;
        return ((T - 1) >> gb_shift(T, static_cast<uint64_t>(e - b))) + 1;
    }
};
// T < 2^32 - 2 for every row, V < 2^27 - 1 (else no bucket index)
__global__ void k_gb_check(const int64_t* __restrict__ rp, const uint64_t* __restrict__ cps, int64_t V,
                           unsigned int* bad) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
        if (rp[v + 1] > rp[v] && cps[rp[v + 1] - 1] >= 0xFFFFFFFEull) atomicOr(bad, 1u);
}
__global__ void k_gb_meta(const int64_t* __restrict__ rp, const uint64_t* __restrict__ cps,
                          const uint64_t* __restrict__ boff, int64_t V, uint4* __restrict__ meta) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = rp[v], e = rp[v + 1];
        const uint64_t T = e > b ? cps[e - 1] : 0;
        meta[v] = make_uint4(static_cast<uint32_t>(boff[v]), T ? gb_shift(T, static_cast<uint64_t>(e - b)) : 0u,
                             static_cast<uint32_t>(T), 0u);
    }
}
// one thread per bucket: its row by a binary search of the bucket offsets, its first region by
// an upper bound of the bucket start in the row's inclusive prefix (the CTPS cache)
__global__ void k_gb_fill(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                          const uint64_t* __restrict__ cps, const uint64_t* __restrict__ boff, int64_t V,
                          uint64_t nbk, const uint4* __restrict__ meta, uint4* __restrict__ gbk) {
    for (uint64_t gi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; gi < nbk; gi += (uint64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = V;   // last v with boff[v] <= gi
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (boff[mid] <= gi) lo = mid; else hi = mid;
        }
        const int64_t v = lo;
        const uint64_t b = gi - boff[v];
        const int64_t rs = rp[v];
        const uint64_t d = static_cast<uint64_t>(rp[v + 1] - rs);
        const uint32_t k = meta[v].y;
        const uint64_t x0 = b << k, x1 = (b + 1) << k;
        uint64_t l = 0, h = d;   // first region with inclusive prefix > x0
        while (l < h) {
            const uint64_t mid = (l + h) >> 1;
            if (cps[rs + mid] <= x0) l = mid + 1; else h = mid;
        }
        uint4* out = gbk + gi * 8;
        uint32_t slot = 0;
        for (uint64_t i = l; i < d && slot < 8; ++i) {
            const uint64_t sx = i ? cps[rs + i - 1] : 0;
            if (sx >= x1) break;
            if (cps[rs + i] == sx) continue;   // empty region: never picked
            if (slot == 7) {   // a 9th region meets the bucket: link entry 7 to the CTPS cache
                uint64_t j = i + 1;
                while (j < d && cps[rs + j] == cps[rs + j - 1]) ++j;
                if (j < d && cps[rs + j - 1] < x1) {
                    const uint64_t ge = static_cast<uint64_t>(rs) + i;
                    out[7] = make_uint4(static_cast<uint32_t>(sx), GB_LINK, static_cast<uint32_t>(ge),
                                        static_cast<uint32_t>(ge >> 32));
                    slot = 8;
                    break;
                }
            }
            const uint32_t u = col[rs + i];
            const uint4 mu = meta[u];
            out[slot++] = make_uint4(static_cast<uint32_t>(sx), u | (mu.y << 27), mu.x, mu.z);
        }
        for (; slot < 8; ++slot) out[slot] = make_uint4(GB_EMPTY, 0u, 0u, 0u);
    }
}

static csaw_status build_gb(csaw_graph* g, int blocks) {
    const int64_t V = g->V;
    if (!g->cps || g->E <= 0 || V >= (int64_t(1) << 27) - 1) return CSAW_OK;
    unsigned int* bad = nullptr;
    uint64_t *boff = nullptr, *part = nullptr;
    auto release = [&]() {
        if (bad) cudaFree(bad);
        if (boff) cudaFree(boff);
        if (part) cudaFree(part);
        cudaGetLastError();
    };
    auto drop = [&]() {   // best-effort: degree walks keep the vertex heads / walk index
        release();
        if (g->gbk) cudaFree(g->gbk);
        if (g->gmeta) cudaFree(g->gmeta);
        g->gbk = nullptr;
        g->gmeta = nullptr;
        g->gb_buckets = 0;
        cudaGetLastError();
        return CSAW_OK;
    };
    if (cudaMalloc(&bad, sizeof(unsigned int)) != cudaSuccess || cudaMalloc(&boff, sizeof(uint64_t) * (V + 1)) != cudaSuccess ||
        cudaMalloc(&part, sizeof(uint64_t) * (SCAN_MAX_GRID + 8)) != cudaSuccess)
        return drop();
    cudaMemset(bad, 0, sizeof(unsigned int));
    k_gb_check<<<blocks, 256>>>(g->row_ptr, g->cps, V, bad);
    unsigned int hb = 0;
    if (cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost) != cudaSuccess || hb) return drop();
    if (device_scan(GbSize{g->row_ptr, g->cps}, static_cast<uint64_t>(V), ScanToArray{boff}, part, nullptr) != CSAW_OK)
        return drop();
    uint64_t nbk = 0;
    if (cudaMemcpy(&nbk, boff + V, sizeof(nbk), cudaMemcpyDeviceToHost) != cudaSuccess) return drop();
    size_t fre = 0, tot = 0;
    if (nbk == 0 || nbk >= (uint64_t(1) << 32) || cudaMemGetInfo(&fre, &tot) != cudaSuccess ||
        nbk * 128 + sizeof(uint4) * V > fre / 2)   // keep half of the free memory for the run
        return drop();
    if (cudaMalloc(&g->gbk, nbk * 128) != cudaSuccess || cudaMalloc(&g->gmeta, sizeof(uint4) * V) != cudaSuccess)
        return drop();
    k_gb_meta<<<blocks, 256>>>(g->row_ptr, g->cps, boff, V, g->gmeta);
    k_gb_fill<<<blocks * 4, 256>>>(g->row_ptr, g->col, g->cps, boff, V, nbk, g->gmeta, g->gbk);
    if (cudaDeviceSynchronize() != cudaSuccess) return drop();
    g->gb_buckets = nbk;
    release();
    return CSAW_OK;
}

// ---------------------------------------------------------------- bucketed walk index, edge weights
// The float path (R28, EdgeBias = w(e)): S_{i+1} = S_i + (double) w_i left to right per row --
// the oracle's order, so S, T and the draw x = r T are the oracle's bit for bit -- cut into
// buckets of width 2^k (k = floor(log2(T / d)) in [-24, 7]); a pick is the last positive-weight
// region with S_i <= x (R28).  A bucket (128 B) lists up to 5 candidate regions: the last
// positive one starting at or before the bucket start, then the positive ones starting inside;
// a 6th turns entry 4 into a link (uk = GB_LINK, T slot = its CSR entry as a u64 bit pattern).
constexpr int GBW_CAP = 5;
constexpr int GBW_KBIAS = 24;
__global__ void k_gbw_prefix(const int64_t* __restrict__ rp, const float* __restrict__ w, int64_t V,
                             double* __restrict__ cpsw, unsigned int* bad) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = rp[v], e = rp[v + 1];
        double S = 0.0;
        for (int64_t i = b; i < e; ++i) {
            S += static_cast<double>(w[i]);
            cpsw[i] = S;
        }
        if (e > b && S > 0.0) {
            const int k = ilogb(S / static_cast<double>(e - b));
            if (k < -GBW_KBIAS || k > 31 - GBW_KBIAS || S * ldexp(1.0, -k) >= 4294967295.0) atomicOr(bad, 1u);
        }
    }
}
struct GbwSize {
    const int64_t* rp;
    const double* cpsw;
    __device__ __forceinline__ uint64_t operator()(uint64_t v) const {
        const int64_t b = rp[v], e = rp[v + 1];
        if (e == b) return 0;
        const double T = cpsw[e - 1];
        if (!(T > 0.0)) return 0;
        const int k = ilogb(T / static_cast<double>(e - b));
        return static_cast<uint64_t>(T * ldexp(1.0, -k)) + 1;   // x = r T <= T: floor(x 2^-k) < nb
    }
};
__global__ void k_gbw_meta(const int64_t* __restrict__ rp, const double* __restrict__ cpsw,
                           const uint64_t* __restrict__ boff, int64_t V, uint4* __restrict__ meta) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = rp[v], e = rp[v + 1];
        const double T = e > b ? cpsw[e - 1] : 0.0;
        const int k = T > 0.0 ? ilogb(T / static_cast<double>(e - b)) : 0;
        const uint64_t tb = static_cast<uint64_t>(__double_as_longlong(T > 0.0 ? T : 0.0));
        meta[v] = make_uint4(static_cast<uint32_t>(boff[v]), static_cast<uint32_t>(k + GBW_KBIAS),
                             static_cast<uint32_t>(tb), static_cast<uint32_t>(tb >> 32));
    }
}
__global__ void k_gbw_fill(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col, const float* __restrict__ w,
                           const double* __restrict__ cpsw, const uint64_t* __restrict__ boff, int64_t V, uint64_t nbk,
                           const uint4* __restrict__ meta, uint8_t* __restrict__ gbw) {
    for (uint64_t gi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; gi < nbk; gi += (uint64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = V;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (boff[mid] <= gi) lo = mid; else hi = mid;
        }
        const int64_t v = lo;
        const uint64_t b = gi - boff[v];
        const int64_t rs = rp[v];
        const int64_t d = rp[v + 1] - rs;
        const int k = static_cast<int>(meta[v].y) - GBW_KBIAS;
        const double x0 = ldexp(static_cast<double>(b), k), x1 = ldexp(static_cast<double>(b + 1), k);
        auto sx = [&](int64_t i) { return i ? cpsw[rs + i - 1] : 0.0; };   // exclusive prefix of region i
        int64_t l = 0, h = d;   // first i with S_excl(i) > x0
        while (l < h) {
            const int64_t mid = (l + h) >> 1;
            if (sx(mid) <= x0) l = mid + 1; else h = mid;
        }
        int64_t r0 = l - 1;   // last positive region starting at or before x0 (exists: S_excl of the first positive one is 0)
        while (r0 > 0 && !(w[rs + r0] > 0.0f)) --r0;
        double* S = reinterpret_cast<double*>(gbw + gi * 128);
        double* Tu = S + GBW_CAP;
        uint32_t* uk = reinterpret_cast<uint32_t*>(Tu + GBW_CAP);
        uint32_t* Bu = uk + GBW_CAP;
        int slot = 0;
        for (int64_t i = r0; i < d && slot < GBW_CAP; ++i) {
            if (i > r0 && (!(w[rs + i] > 0.0f))) continue;
            const double si = sx(i);
            if (i > r0 && si >= x1) break;
            if (slot == GBW_CAP - 1) {   // a further positive region starting inside: link
                int64_t j = i + 1;
                while (j < d && !(w[rs + j] > 0.0f)) ++j;
                if (j < d && sx(j) < x1) {
                    S[slot] = si;
                    Tu[slot] = __longlong_as_double(static_cast<long long>(rs + i));
                    uk[slot] = GB_LINK;
                    Bu[slot] = 0u;
                    slot = GBW_CAP;
                    break;
                }
            }
            const uint32_t u = col[rs + i];
            const uint4 mu = meta[u];
            S[slot] = si;
            Tu[slot] = __longlong_as_double(static_cast<long long>(static_cast<uint64_t>(mu.w) << 32 | mu.z));
            uk[slot] = u | (mu.y << 27);
            Bu[slot] = mu.x;
            ++slot;
        }
        for (; slot < GBW_CAP; ++slot) {
            S[slot] = __longlong_as_double(0x7FF0000000000000ll);   // +inf: never <= x
            Tu[slot] = 0.0;
            uk[slot] = 0u;
            Bu[slot] = 0u;
        }
    }
}

static csaw_status build_gbw(csaw_graph* g, int blocks) {
    const int64_t V = g->V, E = g->E;
    if (!g->w || E <= 0 || V >= (int64_t(1) << 27) - 1) return CSAW_OK;
    unsigned int* bad = nullptr;
    uint64_t *boff = nullptr, *part = nullptr;
    auto release = [&]() {
        if (bad) cudaFree(bad);
        if (boff) cudaFree(boff);
        if (part) cudaFree(part);
        cudaGetLastError();
    };
    auto drop = [&]() {   // best-effort: weighted walks keep the per-step scan (k_walk_vscan<float>)
        release();
        if (g->gbw) cudaFree(g->gbw);
        if (g->gwmeta) cudaFree(g->gwmeta);
        if (g->cpsw) cudaFree(g->cpsw);
        g->gbw = nullptr;
        g->gwmeta = nullptr;
        g->cpsw = nullptr;
        g->gbw_buckets = 0;
        cudaGetLastError();
        return CSAW_OK;
    };
    if (cudaMalloc(&bad, sizeof(unsigned int)) != cudaSuccess || cudaMalloc(&boff, sizeof(uint64_t) * (V + 1)) != cudaSuccess ||
        cudaMalloc(&part, sizeof(uint64_t) * (SCAN_MAX_GRID + 8)) != cudaSuccess ||
        cudaMalloc(&g->cpsw, sizeof(double) * E) != cudaSuccess)
        return drop();
    cudaMemset(bad, 0, sizeof(unsigned int));
    k_gbw_prefix<<<blocks * 4, 64>>>(g->row_ptr, g->w, V, g->cpsw, bad);
    unsigned int hb = 0;
    if (cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost) != cudaSuccess || hb) return drop();
    if (device_scan(GbwSize{g->row_ptr, g->cpsw}, static_cast<uint64_t>(V), ScanToArray{boff}, part, nullptr) != CSAW_OK)
        return drop();
    uint64_t nbk = 0;
    if (cudaMemcpy(&nbk, boff + V, sizeof(nbk), cudaMemcpyDeviceToHost) != cudaSuccess) return drop();
    size_t fre = 0, tot = 0;
    if (nbk == 0 || nbk >= (uint64_t(1) << 32) || cudaMemGetInfo(&fre, &tot) != cudaSuccess ||
        nbk * 128 + sizeof(uint4) * V > fre / 2)
        return drop();
    if (cudaMalloc(&g->gbw, nbk * 128) != cudaSuccess || cudaMalloc(&g->gwmeta, sizeof(uint4) * V) != cudaSuccess)
        return drop();
    k_gbw_meta<<<blocks, 256>>>(g->row_ptr, g->cpsw, boff, V, g->gwmeta);
    k_gbw_fill<<<blocks * 4, 256>>>(g->row_ptr, g->col, g->w, g->cpsw, boff, V, nbk, g->gwmeta, g->gbw);
    if (cudaDeviceSynchronize() != cudaSuccess) return drop();
    g->gbw_buckets = nbk;
    release();
    return CSAW_OK;
}

// ---------------------------------------------------------------- node2vec edge triangle counts
// tri[e] = |N(v) ∩ N(u)| for the CSR entry e = (v -> u): the number of "common
// neighbour" specials of a node2vec step that arrived at v from u (or at u from v), so
// the row total T of the step's CTPS is closed-form (walk.cu k_node2vec_tri).  Built
// once per undirected edge (u > v), written to both entries; any entry without its
// reverse (or a self-loop) marks the graph asymmetric and the cache is not used.
__global__ void k_src_of(const int64_t* __restrict__ rp, int64_t V, uint32_t* __restrict__ src) {
    const int lane = lane_id();
    for (uint64_t v = global_warp_id(); v < static_cast<uint64_t>(V); v += total_warps())
        for (int64_t e = rp[v] + lane; e < rp[v + 1]; e += 32) src[e] = static_cast<uint32_t>(v);
}

// Count of the sorted list small[0, ns) in the sorted list big[0, nb) (warp-collective):
// rows of 32 small entries, the big range of each row narrowed by two 32-ary searches,
// then a per-lane binary search.
__device__ uint32_t warp_intersect_count(const uint32_t* __restrict__ small, uint64_t ns,
                                         const uint32_t* __restrict__ big, uint64_t nb) {
    const int lane = lane_id();
    uint32_t cnt = 0;
    uint64_t lo0 = 0;
    for (uint64_t r0 = 0; r0 < ns && lo0 < nb; r0 += 32) {
        const uint64_t i = r0 + lane;
        const bool valid = i < ns;
        const uint32_t x = valid ? __ldg(small + i) : NONE;
        const uint32_t xmin = __shfl_sync(FULL, x, 0);
        const int last = static_cast<int>(ns - 1 - r0 < 31 ? ns - 1 - r0 : 31);
        const uint32_t xmax = __shfl_sync(FULL, x, last);
        const uint64_t lo = warp_lower_bound(big, lo0, nb, xmin);
        const uint64_t hi = xmax == NONE ? nb : warp_lower_bound(big, lo, nb, xmax + 1u);
        uint64_t l = lo, h = hi;
        while (l < h) {   // same trip count on every lane
            const uint64_t mid = (l + h) >> 1;
            if (__ldg(big + mid) < x) l = mid + 1; else h = mid;
        }
        const bool f = valid && l < hi && __ldg(big + l) == x;
        cnt += __popc(__ballot_sync(FULL, f));
        lo0 = hi;
    }
    return cnt;
}

__global__ void k_tri(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                      const uint32_t* __restrict__ src, int64_t E, uint32_t* __restrict__ tri,
                      unsigned int* __restrict__ asym) {
    for (uint64_t e = global_warp_id(); e < static_cast<uint64_t>(E); e += total_warps()) {
        const uint32_t v = src[e], u = col[e];
        if (u == v) { if (lane_id() == 0) atomicOr(asym, 1u); continue; }
        if (u < v) continue;
        const int64_t bv = rp[v], bu = rp[u];
        const uint64_t dv = static_cast<uint64_t>(rp[v + 1] - bv), du = static_cast<uint64_t>(rp[u + 1] - bu);
        // reverse entry: v in N(u)
        const uint64_t j = warp_lower_bound(col + bu, 0, du, v);
        const bool has_rev = j < du && __ldg(col + bu + j) == v;
        const uint32_t c = dv <= du ? warp_intersect_count(col + bv, dv, col + bu, du)
                                    : warp_intersect_count(col + bu, du, col + bv, dv);
        if (lane_id() == 0) {
            tri[e] = c;
            if (has_rev) tri[bu + j] = c;
            else atomicOr(asym, 1u);
        }
    }
}

// Builds tri (CSAW_GRAPH_N2V_TRI, sorted rows); leaves g->tri null if the graph is not
// symmetric (node2vec then keeps the full-merge kernel).
static csaw_status build_tri(csaw_graph* g, int blocks) {
    if (!g->rows_sorted || g->E <= 0) return CSAW_OK;
    uint32_t* src = nullptr;
    unsigned int* asym = nullptr;
    if (cudaMalloc(&src, sizeof(uint32_t) * g->E) != cudaSuccess || cudaMalloc(&asym, sizeof(unsigned int)) != cudaSuccess ||
        cudaMalloc(&g->tri, sizeof(uint32_t) * g->E) != cudaSuccess) {
        cudaGetLastError();
        if (src) cudaFree(src);
        if (asym) cudaFree(asym);
        if (g->tri) { cudaFree(g->tri); g->tri = nullptr; }
        return CSAW_OK;   // an accelerator: node2vec keeps the merge kernel (csaw_graph_info_t.node2vec_tri = 0)
    }
    cudaMemset(asym, 0, sizeof(unsigned int));
    k_src_of<<<blocks, 256>>>(g->row_ptr, g->V, src);
    k_tri<<<blocks * 4, 256>>>(g->row_ptr, g->col, src, g->E, g->tri, asym);
    unsigned int h = 0;
    const cudaError_t err = cudaMemcpy(&h, asym, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(src);
    cudaFree(asym);
    if (err != cudaSuccess) return fail(CSAW_ERR_CUDA, cudaGetErrorString(err));
    if (h) { cudaFree(g->tri); g->tri = nullptr; }
    return CSAW_OK;
}

// ---------------------------------------------------------------- chunk-total cache (select.cuh)
// For every row of d > TAB candidates: the degree-bias chunk prefix sums build_ctps would
// compute (same chunk size m), then npos, at cc[row start / 64 ...].  Static bias, so
// degree-biased selections read the chunk table instead of scanning the whole pool and
// rescan one chunk per draw (bit-identical).  col may be pinned host memory (OOM modes).
__global__ void k_build_ccache(const int64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                               const uint32_t* __restrict__ deg, int64_t V, uint64_t* __restrict__ cc) {
    const int lane = lane_id();
    for (uint64_t v = global_warp_id(); v < static_cast<uint64_t>(V); v += total_warps()) {
        const int64_t rb = rp[v];
        const uint32_t d = static_cast<uint32_t>(rp[v + 1] - rb);
        if (d <= static_cast<uint32_t>(TAB)) continue;
        const uint32_t nrows = (d + 31) / 32;
        const uint32_t m = ctps_chunk_rows(nrows);
        const uint32_t nch = (nrows + m - 1) / m;
        uint64_t carry = 0;
        uint32_t npos = 0;
        uint64_t* out = cc + static_cast<uint64_t>(rb) / 64;
        for (uint32_t c = 0; c < nch; ++c) {
            const uint32_t e0 = c * m * 32, e1 = min(d, (c + 1) * m * 32);
            uint64_t acc = 0;
            for (uint32_t e = e0 + lane; e < e1; e += 32) {
                const uint32_t b = deg[col[rb + e]];
                acc += b;
                npos += b > 0 ? 1u : 0u;
            }
            carry += warp_sum(acc);
            if (lane == 0) out[c] = carry;
        }
        npos = __reduce_add_sync(FULL, npos);
        if (lane == 0) out[nch] = npos;
    }
}

// Device time of one accelerator build at graph creation (events destroyed on every path).
struct BuildTimer {
    cudaEvent_t c0 = nullptr, c1 = nullptr;
    BuildTimer() {
        if (cudaEventCreate(&c0) != cudaSuccess || cudaEventCreate(&c1) != cudaSuccess) cudaGetLastError();
        if (c0) cudaEventRecord(c0);
    }
    double ms() {
        float t = 0.f;
        if (c1 && cudaEventRecord(c1) == cudaSuccess && cudaEventSynchronize(c1) == cudaSuccess &&
            cudaEventElapsedTime(&t, c0, c1) == cudaSuccess)
            return t;
        cudaGetLastError();
        return 0.0;
    }
    ~BuildTimer() {
        if (c0) cudaEventDestroy(c0);
        if (c1) cudaEventDestroy(c1);
    }
};

static csaw_status build_ccache(csaw_graph* g, const uint32_t* col, int blocks) {
    const uint64_t n = static_cast<uint64_t>(g->E) / 64 + 512;
    if (cudaMalloc(&g->ccache, sizeof(uint64_t) * n) != cudaSuccess) {   // an accelerator: skip it
        cudaGetLastError();
        g->ccache = nullptr;
        return CSAW_OK;
    }
    cudaMemset(g->ccache, 0, sizeof(uint64_t) * n);
    if (g->V > 0) k_build_ccache<<<blocks, 256>>>(g->row_ptr, col, g->deg, g->V, g->ccache);
    g->ccache_entries = n;
    return CSAW_OK;
}
}  // namespace csaw

using namespace csaw;

extern "C" {

CSAW_API const char* csaw_last_error(void) { return g_last_error.c_str(); }

CSAW_API const char* csaw_version(void) { return "csaw-b200 0.1 sm_100a"; }

CSAW_API csaw_status csaw_graph_create(const csaw_csr* csr, const csaw_graph_opts* opt, csaw_graph** out) {
    clear_error();
    if (!csr || !out) return fail(CSAW_ERR_INVALID_ARG, "csr/out is NULL");
    *out = nullptr;
    if (csr->num_vertices < 0 || csr->num_edges < 0) return fail(CSAW_ERR_INVALID_ARG, "negative size");
    if (csr->num_vertices >= static_cast<int64_t>(NONE)) return fail(CSAW_ERR_INVALID_ARG, "num_vertices must be < 2^32-1");
    if (!csr->row_ptr || (csr->num_edges > 0 && !csr->col_idx)) return fail(CSAW_ERR_INVALID_ARG, "row_ptr/col_idx is NULL");
    csaw_graph_opts o{};
    if (opt) o = *opt;
    if (csr->weights && o.device_budget_bytes > 0)
        return fail(CSAW_ERR_UNSUPPORTED, "edge weights are not supported in out-of-memory mode");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(CSAW_ERR_CUDA, "no CUDA device: the C-SAW library has no CPU fallback");
    }
    if (o.device < 0 || o.device >= ndev) return fail(CSAW_ERR_INVALID_ARG, "bad device ordinal");
    CSAW_CUDA(cudaSetDevice(o.device));

    csaw_graph* g = new csaw_graph();
    g->device = o.device;
    g->V = csr->num_vertices;
    g->E = csr->num_edges;
    cudaDeviceProp prop;
    CSAW_CUDA(cudaGetDeviceProperties(&prop, o.device));
    g->num_sms = prop.multiProcessorCount;
    g->oom = o.device_budget_bytes > 0;
    g->force_batched = (o.flags & CSAW_GRAPH_SAMPLE_BATCHED) != 0;
    g->flags = o.flags;
    const int64_t V = g->V, E = g->E;
    ValidateOut* dv = nullptr;
    uint32_t* dcol = nullptr;
    auto cleanup = [&](csaw_status s) {
        if (dv) cudaFree(dv);
        if (dcol && dcol != g->col) cudaFree(dcol);
        csaw_graph_destroy(g);
        return s;
    };
#define CREATE_CUDA(call, what)                                                          \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) return cleanup(cuda_fail(e_, what, __FILE__, __LINE__));  \
    } while (0)
    CREATE_CUDA(cudaMalloc(&g->row_ptr, sizeof(int64_t) * (V + 1)), "cudaMalloc(row_ptr)");
    CREATE_CUDA(cudaMalloc(&g->deg, sizeof(uint32_t) * std::max<int64_t>(V, 1)), "cudaMalloc(deg)");
    CREATE_CUDA(cudaMemcpy(g->row_ptr, csr->row_ptr, sizeof(int64_t) * (V + 1), cudaMemcpyDefault), "copy row_ptr");
    int64_t rp_first = -1, rp_last = -1;
    cudaMemcpy(&rp_first, g->row_ptr, sizeof(int64_t), cudaMemcpyDeviceToHost);
    cudaMemcpy(&rp_last, g->row_ptr + V, sizeof(int64_t), cudaMemcpyDeviceToHost);
    if (rp_first != 0 || rp_last != E)
        return cleanup(fail(CSAW_ERR_BAD_GRAPH, "row_ptr[0] must be 0 and row_ptr[V] must equal num_edges"));
    CREATE_CUDA(cudaMalloc(&dv, sizeof(ValidateOut)), "cudaMalloc");
    ValidateOut hv{~0ull, ~0ull, 0, 0, 0, ~0ull};
    cudaMemcpy(dv, &hv, sizeof(hv), cudaMemcpyHostToDevice);
    const int blocks = g->num_sms * 8;
    if (V > 0) k_validate_rows<<<blocks, 256>>>(g->row_ptr, V, g->deg, dv);
    CREATE_CUDA(cudaMemcpy(&hv, dv, sizeof(hv), cudaMemcpyDeviceToHost), "validate rows");
    if (hv.bad_rowptr != ~0ull)
        return cleanup(fail(CSAW_ERR_BAD_GRAPH, "row_ptr decreases at vertex " + std::to_string(hv.bad_rowptr - 1)));
    g->max_deg = static_cast<int64_t>(hv.max_deg);
    g->nonisolated = static_cast<int64_t>(hv.nonisolated);
    if (g->max_deg >= static_cast<int64_t>(NONE) - 64)
        return cleanup(fail(CSAW_ERR_UNSUPPORTED, "max degree must be < 2^32-64"));

    if (!g->oom) {
        CREATE_CUDA(cudaMalloc(&dcol, sizeof(uint32_t) * std::max<int64_t>(E, 1)), "cudaMalloc(col)");
        g->col = dcol;
        if (E > 0) CREATE_CUDA(cudaMemcpy(dcol, csr->col_idx, sizeof(uint32_t) * E, cudaMemcpyDefault), "copy col_idx");
        if (E > 0) k_validate_cols<<<blocks, 256>>>(dcol, E, 0, V, dv);
        if (V > 0) k_validate_sorted<<<blocks, 256>>>(g->row_ptr, dcol, 0, V, dv);
        if (csr->weights) {   // EdgeBias = w(e): fp32, finite, >= 0; VROW entries of zero padding (vscan.cuh)
            CREATE_CUDA(cudaMalloc(&g->w, sizeof(float) * (E + VSCAN_PAD)), "cudaMalloc(weights)");
            CREATE_CUDA(cudaMemset(g->w, 0, sizeof(float) * (E + VSCAN_PAD)), "memset(weights)");
            if (E > 0) CREATE_CUDA(cudaMemcpy(g->w, csr->weights, sizeof(float) * E, cudaMemcpyDefault), "copy weights");
            if (E > 0) k_validate_weights<<<blocks, 256>>>(g->w, E, dv);
        }
    } else {
        // Out-of-memory mode (§5): the full col_idx lives in pinned host memory; the
        // device holds row_ptr + deg and R arena slots of one partition each.  The
        // CSR is validated slice by slice through slot 0, so the device never holds
        // more than the budget.
        auto& st = g->oomst;
        st.budget = o.device_budget_bytes;
        st.zerocopy = (o.flags & CSAW_GRAPH_OOM_ZEROCOPY) != 0;
        st.ws = (o.flags & CSAW_GRAPH_OOM_NO_WS) == 0;
        st.bal = (o.flags & CSAW_GRAPH_OOM_NO_BAL) == 0;
        st.P = o.num_partitions > 0 ? o.num_partitions : 4;
        st.R = o.max_resident > 0 ? o.max_resident : 2;
        st.S = o.num_streams > 0 ? o.num_streams : 2;
        if (st.P > V && V > 0) st.P = static_cast<int32_t>(V);
        if (st.P < 1) st.P = 1;
        if (st.R > st.P) st.R = st.P;
        CREATE_CUDA(cudaMallocHost(&st.h_row, sizeof(int64_t) * (V + 1)), "cudaMallocHost(row)");
        cudaMemcpy(st.h_row, g->row_ptr, sizeof(int64_t) * (V + 1), cudaMemcpyDeviceToHost);
        // equal contiguous vertex ranges, remainder to the lowest partitions (R23)
        st.bounds.assign(st.P + 1, 0);
        const int64_t base = V / st.P, rem = V % st.P;
        for (int p = 0; p < st.P; ++p) st.bounds[p + 1] = st.bounds[p] + base + (p < rem ? 1 : 0);
        st.ebeg.assign(st.P + 1, 0);
        int64_t maxpe = 0;
        for (int p = 0; p <= st.P; ++p) st.ebeg[p] = st.h_row[st.bounds[p]];
        for (int p = 0; p < st.P; ++p) maxpe = std::max(maxpe, st.ebeg[p + 1] - st.ebeg[p]);
        st.slot_edges = std::max<int64_t>(maxpe, 1);
        // + the chunk-total cache of the degree bias when it fits (E / 64 + 512 u64)
        const int64_t cc_bytes = static_cast<int64_t>(sizeof(uint64_t)) * (E / 64 + 512);
        const int64_t base_resident = sizeof(int64_t) * (V + 1) + sizeof(uint32_t) * V;
        const int64_t arena0 = static_cast<int64_t>(st.zerocopy ? 1 : st.R) * st.slot_edges *
                               static_cast<int64_t>(sizeof(uint32_t));
        st.want_ccache = !(o.flags & CSAW_GRAPH_OOM_NO_CHUNK_CACHE) && base_resident + cc_bytes + arena0 <= st.budget;
        const int64_t resident_bytes = base_resident + (st.want_ccache ? cc_bytes : 0);
        // the arena holds R partitions; zero-copy mode validates through a 1-partition slot only
        const int64_t arena = static_cast<int64_t>(st.zerocopy ? 1 : st.R) * st.slot_edges *
                              static_cast<int64_t>(sizeof(uint32_t));
        if (resident_bytes + arena > st.budget)
            return cleanup(fail(CSAW_ERR_NO_MEMORY,
                                "OOM mode: row_ptr+deg (" + std::to_string(resident_bytes) + " B) + " +
                                    std::to_string(st.R) + " partition slots (" + std::to_string(arena) +
                                    " B) exceed the device budget " + std::to_string(st.budget) + " B"));
        CREATE_CUDA(cudaMalloc(&st.d_slots, arena), "cudaMalloc(arena)");
        if (o.flags & CSAW_GRAPH_OOM_PEER_STORE) {   // partition store in a peer GPU's HBM (NEXT-4(i))
            if (o.store_device < 0 || o.store_device >= ndev)
                return cleanup(fail(CSAW_ERR_INVALID_ARG, "OOM peer store: bad store_device"));
            st.store_device = o.store_device;
            if (o.store_device != o.device) {
                int can = 0;
                CREATE_CUDA(cudaDeviceCanAccessPeer(&can, o.device, o.store_device), "peer query");
                if (!can) return cleanup(fail(CSAW_ERR_UNSUPPORTED, "OOM peer store: no peer access to store_device"));
                const cudaError_t pe = cudaDeviceEnablePeerAccess(o.store_device, 0);
                if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CREATE_CUDA(pe, "enable peer access");
                cudaGetLastError();
            }
            CREATE_CUDA(cudaSetDevice(o.store_device), "cudaSetDevice(store)");
            const cudaError_t me = cudaMalloc(&st.d_store, sizeof(uint32_t) * std::max<int64_t>(E, 1));
            cudaError_t ce = cudaSuccess;
            if (me == cudaSuccess && E > 0) ce = cudaMemcpy(st.d_store, csr->col_idx, sizeof(uint32_t) * E, cudaMemcpyDefault);
            CREATE_CUDA(cudaSetDevice(o.device), "cudaSetDevice");
            CREATE_CUDA(me, "cudaMalloc(peer store)");
            CREATE_CUDA(ce, "copy col_idx to the peer store");
            st.src_col = st.d_store;
        } else {
            CREATE_CUDA(cudaMallocHost(&st.h_col, sizeof(uint32_t) * std::max<int64_t>(E, 1)), "cudaMallocHost(col)");
            if (E > 0) CREATE_CUDA(cudaMemcpy(st.h_col, csr->col_idx, sizeof(uint32_t) * E, cudaMemcpyDefault), "copy col_idx");
            st.src_col = st.h_col;
        }
        for (int p = 0; p < st.P; ++p) {
            const int64_t e0 = st.ebeg[p], ne = st.ebeg[p + 1] - e0;
            if (ne == 0) continue;
            CREATE_CUDA(cudaMemcpy(st.d_slots, st.src_col + e0, sizeof(uint32_t) * ne, cudaMemcpyDefault), "slice");
            k_validate_cols<<<blocks, 256>>>(st.d_slots, ne, e0, V, dv);
            k_validate_sorted<<<blocks, 256>>>(g->row_ptr, st.d_slots - e0, st.bounds[p], st.bounds[p + 1], dv);
            CREATE_CUDA(cudaDeviceSynchronize(), "validate slice");
        }
        st.resident.assign(st.R, -1);
        if (st.zerocopy) {   // no partition staging: release the validation slot
            cudaFree(st.d_slots);
            st.d_slots = nullptr;
            // Resident prefix of col_idx filling the budget left after row_ptr + deg and a
            // run-state reserve (walk pools, outputs, scratch: min(512 MiB, budget / 8)).  A walk step that reads entry e
            // takes it from the device when e < colc_n, else from pinned host memory.  For
            // MDRW every entry is equally likely to be read (a row is picked with probability
            // proportional to its degree, then one of its entries uniformly), so the fraction
            // of host reads is the uncached fraction, whichever entries are cached.
            const int64_t reserve = std::min<int64_t>(int64_t(512) << 20, st.budget / 8);
            const int64_t room = st.budget - resident_bytes - reserve;
            st.colc_n = (o.flags & CSAW_GRAPH_OOM_ZC_NO_PREFIX) || room <= 0 ? 0 : std::min<int64_t>(E, room / 4);
            if (st.colc_n > 0) {
                if (cudaMalloc(&st.d_colc, sizeof(uint32_t) * st.colc_n) != cudaSuccess) {
                    cudaGetLastError();
                    st.d_colc = nullptr;
                    st.colc_n = 0;
                } else {
                    CREATE_CUDA(cudaMemcpy(st.d_colc, st.src_col, sizeof(uint32_t) * st.colc_n, cudaMemcpyDefault),
                                "copy resident col prefix");
                }
            }
        }
        st.streams.resize(st.S);
        for (auto& s : st.streams) CREATE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    }
    CREATE_CUDA(cudaMemcpy(&hv, dv, sizeof(hv), cudaMemcpyDeviceToHost), "validate");
    cudaFree(dv);
    dv = nullptr;
    if (hv.bad_col != ~0ull)
        return cleanup(fail(CSAW_ERR_BAD_GRAPH, "col_idx[" + std::to_string(hv.bad_col - 1) + "] >= num_vertices"));
    if (hv.bad_weight != ~0ull)
        return cleanup(fail(CSAW_ERR_BAD_GRAPH, "weights[" + std::to_string(hv.bad_weight - 1) +
                                                    "] is negative or not finite"));
    g->rows_sorted = hv.unsorted == 0;
    // chunk-total cache of the degree bias: always in OOM mode when it fits the budget (no
    // per-entry cache does), on request in memory
    if ((g->oom && g->oomst.want_ccache) || (!g->oom && (o.flags & CSAW_GRAPH_CHUNK_CACHE))) {
        const csaw_status cs_ = build_ccache(g, g->oom ? g->oomst.src_col : g->col, blocks);
        if (cs_ != CSAW_OK) return cleanup(cs_);
    }
    // Accelerators.  The CTPS cache is the one structure a caller asks for by name and is
    // mandatory (NO_MEMORY if it does not fit); everything else -- walk index and heads,
    // next-vertex metadata, node2vec index / triangle counts, materialised edge bias, chunk
    // totals -- is best-effort: without memory for it the graph is created without it
    // (csaw_graph_info_t says what was built) and the selections use the general kernels.
    if ((o.flags & CSAW_GRAPH_CTPS_CACHE) && !g->oom) {
        BuildTimer tm;
        CREATE_CUDA(cudaMalloc(&g->cps, sizeof(uint64_t) * std::max<int64_t>(E, 1)), "cudaMalloc(cps)");
        CREATE_CUDA(cudaMalloc(&g->npos, sizeof(uint32_t) * std::max<int64_t>(V, 1)), "cudaMalloc(npos)");
        if (V > 0) k_build_cps<<<blocks, 256>>>(g->row_ptr, g->col, g->deg, V, g->cps, g->npos);
        // B-tree index over the cached prefix: dense segments (prefix sum of the sizes)
        CREATE_CUDA(cudaMalloc(&g->bt_off, sizeof(uint64_t) * (V + 1)), "cudaMalloc(bt_off)");
        uint64_t* part = nullptr;
        CREATE_CUDA(cudaMalloc(&part, sizeof(uint64_t) * (SCAN_MAX_GRID + 8)), "cudaMalloc");
        device_scan(BtSize{g->row_ptr}, static_cast<uint64_t>(V), ScanToArray{g->bt_off}, part, nullptr);
        uint64_t btn = 0;
        const cudaError_t be = cudaMemcpy(&btn, g->bt_off + V, sizeof(uint64_t), cudaMemcpyDeviceToHost);
        cudaFree(part);
        CREATE_CUDA(be, "bt size");
        CREATE_CUDA(cudaMalloc(&g->bt, sizeof(uint64_t) * std::max<uint64_t>(btn, 1)), "cudaMalloc(bt)");
        if (V > 0) k_build_bt<<<blocks, 256>>>(g->row_ptr, g->cps, g->bt_off, V, g->bt);
        // (next-vertex metadata for k_walk_cached: CSAW_GRAPH_NEXT_META, below; measured 2.5 %
        // slower on cfg2 -- the extra 256 B per step outweighs the saved row_ptr round)
        if (!(o.flags & CSAW_GRAPH_NO_WALK_INDEX)) {
            const csaw_status ws = build_wix(g, blocks);
            if (ws != CSAW_OK) return cleanup(ws);
        }
        if (o.flags & CSAW_GRAPH_WALK_BUCKETS) {
            const csaw_status gs = build_gb(g, blocks);
            if (gs != CSAW_OK) return cleanup(gs);
        }
        g->cache_build_ms = tm.ms();
    }
    if ((o.flags & CSAW_GRAPH_NEXT_META) && !g->oom && !g->nmp && g->max_deg < (1 << 24) && E < (int64_t(1) << 40) &&
        E > 0) {   // nmp[e] = row_ptr[col[e]] << 24 | deg(col[e]) (MDRW: k_mdrw_fast)
        BuildTimer tm;
        if (cudaMalloc(&g->nmp, sizeof(uint64_t) * E) == cudaSuccess) k_build_nmp<<<blocks, 256>>>(g->row_ptr, g->col, E, g->nmp);
        else { cudaGetLastError(); g->nmp = nullptr; }
        if (g->nmp) g->cache_build_ms += tm.ms();
    }
    if ((o.flags & CSAW_GRAPH_NEXT_RECORD) && !g->oom && !g->nrec && E > 0) {   // best-effort (MDRW: k_mdrw_fast)
        BuildTimer tm;
        if (cudaMalloc(&g->nrec, sizeof(uint4) * E) == cudaSuccess) k_build_nrec<<<blocks, 256>>>(g->row_ptr, g->col, E, g->nrec);
        else { cudaGetLastError(); g->nrec = nullptr; }
        if (g->nrec) g->cache_build_ms += tm.ms();
    }
    if ((o.flags & CSAW_GRAPH_N2V_INDEX) && !g->oom) {   // node2vec per-edge intersection index (n2v_index.cu)
        BuildTimer tm;
        const csaw_status xs = build_n2v_index(g, blocks);
        const double ms = tm.ms();
        if (xs != CSAW_OK) return cleanup(xs);
        g->cache_build_ms += ms;
    }
    if ((o.flags & CSAW_GRAPH_N2V_TRI) && !g->oom && !g->n2x_rec) {   // node2vec edge triangle counts (k_node2vec_tri; not needed with the index)
        BuildTimer tm;
        const csaw_status ts = build_tri(g, blocks);
        const double ms = tm.ms();
        if (ts != CSAW_OK) return cleanup(ts);
        g->cache_build_ms += ms;
    }
    if ((o.flags & CSAW_GRAPH_EDGE_BIAS) && !g->oom) {   // ebias[e] = deg(col[e]) (vscan.cuh degree pools)
        BuildTimer tm;
        if (cudaMalloc(&g->ebias, sizeof(uint32_t) * (E + VSCAN_PAD)) != cudaSuccess) {
            cudaGetLastError();
            g->ebias = nullptr;
        } else {
            cudaMemsetAsync(g->ebias, 0, sizeof(uint32_t) * (E + VSCAN_PAD));
            if (E > 0) k_build_ebias<<<blocks, 256>>>(g->col, g->deg, E, g->ebias);
        }
        const double ms = tm.ms();
        if (g->ebias) g->cache_build_ms += ms;
    }
    if ((o.flags & CSAW_GRAPH_WALK_BUCKETS) && g->w && !g->oom) {   // weighted walks: fp64 bucketed index
        BuildTimer tm;
        const csaw_status ws = build_gbw(g, blocks);
        const double ms = tm.ms();
        if (ws != CSAW_OK) return cleanup(ws);
        if (g->gbw) g->cache_build_ms += ms;
    }
    CREATE_CUDA(cudaEventCreate(&g->ev0), "event");
    CREATE_CUDA(cudaEventCreate(&g->ev1), "event");
    CREATE_CUDA(cudaEventCreateWithFlags(&g->ev_done, cudaEventDisableTiming), "event");
    CREATE_CUDA(cudaDeviceSynchronize(), "graph_create");
#undef CREATE_CUDA
    *out = g;
    return CSAW_OK;
}

CSAW_API csaw_status csaw_graph_destroy(csaw_graph* g) {
    if (!g) return CSAW_OK;
    cudaSetDevice(g->device);
    cudaDeviceSynchronize();
    if (g->row_ptr) cudaFree(g->row_ptr);
    if (g->col) cudaFree(g->col);
    if (g->deg) cudaFree(g->deg);
    if (g->cps) cudaFree(g->cps);
    if (g->npos) cudaFree(g->npos);
    if (g->bt) cudaFree(g->bt);
    if (g->bt_off) cudaFree(g->bt_off);
    if (g->nmp) cudaFree(g->nmp);
    if (g->nrec) cudaFree(g->nrec);
    if (g->gbk) cudaFree(g->gbk);
    if (g->gmeta) cudaFree(g->gmeta);
    if (g->gbw) cudaFree(g->gbw);
    if (g->gwmeta) cudaFree(g->gwmeta);
    if (g->cpsw) cudaFree(g->cpsw);
    if (g->c32) cudaFree(g->c32);
    if (g->ccache) cudaFree(g->ccache);
    if (g->whead) cudaFree(g->whead);
    if (g->tri) cudaFree(g->tri);
    if (g->n2x_rec) cudaFree(g->n2x_rec);
    if (g->n2x_idx) cudaFree(g->n2x_idx);
    if (g->wcol) cudaFree(g->wcol);
    if (g->w) cudaFree(g->w);
    if (g->ebias) cudaFree(g->ebias);
    if (g->winn) cudaFree(g->winn);
    auto& st = g->oomst;
    if (st.h_col) cudaFreeHost(st.h_col);
    if (st.d_store) {
        cudaSetDevice(st.store_device);
        cudaFree(st.d_store);
        cudaSetDevice(g->device);
    }
    if (st.h_row) cudaFreeHost(st.h_row);
    if (st.d_slots) cudaFree(st.d_slots);
    if (st.d_colc) cudaFree(st.d_colc);
    for (auto s : st.streams) cudaStreamDestroy(s);
    if (g->ev0) cudaEventDestroy(g->ev0);
    if (g->ev1) cudaEventDestroy(g->ev1);
    if (g->ev_done) cudaEventDestroy(g->ev_done);
    if (g->copy_st) cudaStreamDestroy(g->copy_st);
    for (cudaEvent_t e : g->copy_ev) if (e) cudaEventDestroy(e);
    g->scratch.release_all();
    delete g;
    return CSAW_OK;
}

CSAW_API csaw_status csaw_graph_info(const csaw_graph* g, csaw_graph_info_t* out) {
    clear_error();
    if (!g || !out) return fail(CSAW_ERR_INVALID_ARG, "graph/out is NULL");
    out->num_vertices = g->V;
    out->num_edges = g->E;
    out->max_degree = g->max_deg;
    out->nonisolated = g->nonisolated;
    out->rows_sorted = g->rows_sorted;
    out->oom_mode = g->oom ? 1 : 0;
    out->device_bytes = sizeof(int64_t) * (g->V + 1) + sizeof(uint32_t) * g->V +
                        (g->col ? sizeof(uint32_t) * g->E : 0) + static_cast<int64_t>(g->scratch.bytes_held()) +
                        (g->oom ? (g->oomst.zerocopy ? 0 : static_cast<int64_t>(g->oomst.R) * g->oomst.slot_edges * 4) +
                                      g->oomst.colc_n * 4 : 0) +
                        (g->cps ? static_cast<int64_t>(sizeof(uint64_t) * g->E + sizeof(uint32_t) * g->V) : 0) +
                        (g->wix_leaf ? static_cast<int64_t>(sizeof(uint32_t) * (2 * g->wleaf_entries + g->winn_entries) + sizeof(uint4) * g->V) : 0) +
                        (g->whead ? static_cast<int64_t>(sizeof(uint32_t)) * WIX_HEAD_WORDS * g->V : 0) +
                        (g->tri ? static_cast<int64_t>(sizeof(uint32_t) * g->E) : 0) +
                        (g->n2x_rec ? static_cast<int64_t>(N2X_U4 * sizeof(uint4) * g->E + sizeof(uint32_t) * g->n2x_total) : 0) +
                        (g->nmp ? static_cast<int64_t>(sizeof(uint64_t) * g->E) : 0) +
                        (g->nrec ? static_cast<int64_t>(sizeof(uint4) * g->E) : 0) +
                        (g->gbk ? static_cast<int64_t>(128 * g->gb_buckets + sizeof(uint4) * g->V) : 0) +
                        (g->gbw ? static_cast<int64_t>(128 * g->gbw_buckets + sizeof(uint4) * g->V + sizeof(double) * g->E) : 0) +
                        (g->w ? static_cast<int64_t>(sizeof(float) * (g->E + VSCAN_PAD)) : 0) +
                        (g->ebias ? static_cast<int64_t>(sizeof(uint32_t) * (g->E + VSCAN_PAD)) : 0) +
                        static_cast<int64_t>(sizeof(uint64_t) * g->ccache_entries);
    out->ctps_cache = g->cps ? 1 : 0;
    out->walk_index_leaf = g->wix_leaf;
    out->walk_index_group = g->wix_leaf ? g->wix_group : 0;
    out->node2vec_tri = g->tri ? 1 : 0;
    out->walk_index_heads = g->whead ? 1 : 0;
    out->node2vec_index = g->n2x_rec ? 1 : 0;
    out->cache_build_ms = g->cache_build_ms;
    out->has_weights = g->w ? 1 : 0;
    out->edge_bias = g->ebias ? 1 : 0;
    out->walk_buckets = (g->gbk ? 1 : 0) | (g->gbw ? 2 : 0);
    return CSAW_OK;
}

CSAW_API csaw_status csaw_stats(const csaw_graph* g, csaw_run_stats* out) {
    clear_error();
    if (!g || !out) return fail(CSAW_ERR_INVALID_ARG, "graph/out is NULL");
    CSAW_CUDA(cudaSetDevice(g->device));
    CSAW_CUDA(cudaEventSynchronize(g->ev1));
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, g->ev0, g->ev1) == cudaSuccess) g->stats.kernel_ms = ms;
    else cudaGetLastError();
    double hot = 0.0;
    for (int i = 0; i < g->hot_used; ++i) {
        float h = 0.f;
        if (cudaEventElapsedTime(&h, g->hot_ev[2 * i], g->hot_ev[2 * i + 1]) == cudaSuccess) hot += h;
        else cudaGetLastError();
    }
    g->stats.hot_kernel_ms = hot;
    if (g->pending_counters) {
        unsigned long long c[4] = {0, 0, 0, 0};
        CSAW_CUDA(cudaMemcpy(c, g->pending_counters, sizeof(c), cudaMemcpyDeviceToHost));
        g->stats.neighbours_scanned = c[0];
        g->stats.pools = c[1];
        g->stats.cache_probes = c[2];
        g->stats.index_bytes = c[3];
        g->pending_counters = nullptr;
    }
    *out = g->stats;
    return CSAW_OK;
}

CSAW_API csaw_status csaw_sample_capacity(const csaw_bias* bias, const int32_t* fanout, int32_t depth,
                                          int64_t n, int64_t* cap) {
    clear_error();
    if (!bias || !cap || n < 0 || depth < 0) return fail(CSAW_ERR_INVALID_ARG, "bad argument");
    double total = 0;
    if (bias->kind == CSAW_BIAS_SNOWBALL) {
        // unbounded (a BFS ball): a first guess; csaw_sample reports the exact size on CAPACITY
        total = 64.0 * n * depth + 1024;
    } else if (bias->kind == CSAW_BIAS_FOREST_FIRE) {
        // mean burn count pf/(1-pf) per expanded vertex; 4x headroom + slack
        const double m = bias->pf / std::max(1e-9, 1.0 - bias->pf);
        double level = 1.0;
        for (int d = 0; d < depth; ++d) { level *= m; total += level; }
        total = 4.0 * total * n + 1024;
    } else if (bias->kind == CSAW_BIAS_LAYER) {
        if (!fanout) return fail(CSAW_ERR_INVALID_ARG, "fanout is NULL");
        for (int d = 0; d < depth; ++d) total += fanout[d];
        total *= n;
    } else {
        if (!fanout) return fail(CSAW_ERR_INVALID_ARG, "fanout is NULL");
        double level = 1.0;
        for (int d = 0; d < depth; ++d) { level *= fanout[d]; total += level; }
        total *= n;
    }
    *cap = total > 9.0e18 ? INT64_MAX : static_cast<int64_t>(total);
    return CSAW_OK;
}

static csaw_status check_bias(const csaw_bias* b) {
    if (!b) return fail(CSAW_ERR_INVALID_ARG, "bias is NULL");
    if (b->kind < CSAW_BIAS_UNIFORM || b->kind > CSAW_BIAS_WEIGHT) return fail(CSAW_ERR_INVALID_ARG, "unknown bias kind");
    if (b->migration < 0 || b->migration > 2) return fail(CSAW_ERR_INVALID_ARG, "migration must be 0, 1 or 2");
    if (b->a_max != 0 && (b->a_max < 2 || b->a_max > 16382 || (b->a_max & 1)))
        return fail(CSAW_ERR_INVALID_ARG, "a_max must be 0 (default 64) or even in [2, 16382]");
    return CSAW_OK;
}

// Any seed >= V sets *bad (a plain store into pinned, host-mapped memory).
__global__ void k_check_seeds(const uint32_t* __restrict__ seeds, int64_t n, int64_t V, volatile unsigned* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (static_cast<int64_t>(seeds[i]) >= V) *bad = 1u;
}

CSAW_API csaw_status csaw_walk(const csaw_graph* g, const csaw_bias* bias, int32_t length, const uint32_t* seeds,
                               int64_t n, uint64_t instance_base, uint64_t rng_seed, uint32_t* path, void* stream) {
    CSAW_TRY(begin_call(g));
    CSAW_TRY(check_bias(bias));
    const csaw_bias b = *bias;
    if (b.kind == CSAW_BIAS_FOREST_FIRE || b.kind == CSAW_BIAS_LAYER || b.kind == CSAW_BIAS_SNOWBALL)
        return fail(CSAW_ERR_INVALID_ARG, "forest fire / layer / snowball are sampling selectors (use csaw_sample)");
    if (length < 0 || n < 0) return fail(CSAW_ERR_INVALID_ARG, "negative length / n_walkers");
    if (b.kind == CSAW_BIAS_NODE2VEC && !(b.p > 0 && b.q > 0 && std::isfinite(b.p) && std::isfinite(b.q)))
        return fail(CSAW_ERR_INVALID_ARG, "node2vec needs finite p, q > 0");
    if (b.kind == CSAW_BIAS_MDRW && b.pool_size < 1) return fail(CSAW_ERR_INVALID_ARG, "MDRW needs pool_size >= 1");
    if ((b.kind == CSAW_BIAS_RESTART || b.kind == CSAW_BIAS_JUMP) && !(b.pf >= 0.0 && b.pf < 1.0))
        return fail(CSAW_ERR_INVALID_ARG, "restart / jump probability (pf) must be in [0, 1)");
    if (instance_base + static_cast<uint64_t>(n) > 0xFFFFFFFFull)
        return fail(CSAW_ERR_INVALID_ARG, "instance ids must fit in 32 bits");
    if (n == 0 || (b.kind != CSAW_BIAS_MDRW && length < 0)) return CSAW_OK;
    if (!seeds || !path) return fail(CSAW_ERR_INVALID_ARG, "seeds/path is NULL");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t nseeds = b.kind == CSAW_BIAS_MDRW ? n * static_cast<int64_t>(b.pool_size) : n;
    const int64_t nout = b.kind == CSAW_BIAS_MDRW ? n * static_cast<int64_t>(length) * 2
                                                  : n * (static_cast<int64_t>(length) + 1);
    const PtrKind ks = ptr_kind(seeds, g->device), kp = ptr_kind(path, g->device);
    if (ks == PtrKind::OtherDevice || kp == PtrKind::OtherDevice)
        return fail(CSAW_ERR_INVALID_ARG, "seeds/path live on another GPU than the graph");
    const bool seeds_dev = ks == PtrKind::Device;
    const bool path_dev = kp == PtrKind::Device;
    CallOrder order(g, st);
    const uint32_t* d_seeds = seeds;
    uint32_t* d_path = path;
    if (!seeds_dev) {
        void* p;
        CSAW_TRY(g->scratch.get(SL_SEEDS, sizeof(uint32_t) * nseeds, &p));
        CSAW_CUDA(cudaMemcpyAsync(p, seeds, sizeof(uint32_t) * nseeds, cudaMemcpyHostToDevice, st));
        d_seeds = static_cast<const uint32_t*>(p);
    }
    // seeds must be vertices: checked on the device before any walk kernel reads a row
    {
        void* hm;
        CSAW_TRY(g->pinned.get(4096, &hm));
        volatile unsigned* bad = static_cast<volatile unsigned*>(hm) + 1000;
        *bad = 0u;
        const int cb = static_cast<int>(std::min<int64_t>((nseeds + 255) / 256, int64_t(g->num_sms) * 8));
        k_check_seeds<<<std::max(cb, 1), 256, 0, st>>>(d_seeds, nseeds, g->V, bad);
        note_launch();
        CSAW_CUDA(cudaGetLastError());
        CSAW_CUDA(cudaStreamSynchronize(st));
        if (*bad) return fail(CSAW_ERR_OUT_OF_RANGE, "a seed vertex is >= num_vertices");
    }
    // pinned host output: the kernels write the paths straight into it over the host link,
    // overlapped with the walk (no device staging, no copy after the kernel)
    // (kernels that store one scattered 4 B entry per thread and step -- the node2vec index
    // kernel -- would turn that into uncoalesced host-link writes: they stage and copy)
    void* const path_pinned = (path_dev || !walk_path_direct_ok(g, b)) ? nullptr : pinned_device_ptr(path);
    if (path_pinned) {
        d_path = static_cast<uint32_t*>(path_pinned);
    } else if (!path_dev) {
        void* p;
        CSAW_TRY(g->scratch.get(SL_OUT, sizeof(uint32_t) * std::max<int64_t>(nout, 1), &p));
        d_path = static_cast<uint32_t*>(p);
    }
    csaw_status s;
    bool copied = false;
    if (g->oom && g->oomst.zerocopy) {
        s = run_walk(g, b, length, d_seeds, n, instance_base, rng_seed, d_path, st);   // every kernel reads src_col
    } else if (g->oom) {
        if (b.kind == CSAW_BIAS_MDRW) s = run_mdrw_oom(g, b, length, d_seeds, n, instance_base, rng_seed, d_path, st);
        else s = run_walk_oom(g, b, length, d_seeds, n, instance_base, rng_seed, d_path, st);
    } else {
        // a pinned host path the kernel cannot write directly: run_walk may copy it back itself,
        // chunk by chunk behind the walk
        uint32_t* h_pipe = (!path_dev && !path_pinned && kp == PtrKind::Pinned) ? path : nullptr;
        s = run_walk(g, b, length, d_seeds, n, instance_base, rng_seed, d_path, st, h_pipe, &copied);
    }
    if (s != CSAW_OK) return s;
    if (!path_dev && !path_pinned && !copied) {
        CSAW_CUDA(cudaMemcpyAsync(path, d_path, sizeof(uint32_t) * nout, cudaMemcpyDeviceToHost, st));
    }
    if (!seeds_dev || !path_dev) CSAW_CUDA(cudaStreamSynchronize(st));
    return CSAW_OK;
}

CSAW_API csaw_status csaw_sample(const csaw_graph* g, const csaw_bias* bias, const int32_t* fanout, int32_t depth,
                                 const uint32_t* seeds, int64_t n, uint64_t instance_base, uint64_t rng_seed,
                                 uint64_t* offsets, uint32_t* src, uint32_t* dst, uint8_t* edge_depth,
                                 int64_t capacity, int64_t* num_edges, void* stream) {
    CSAW_TRY(begin_call(g));
    CSAW_TRY(check_bias(bias));
    const csaw_bias b = *bias;
    if (b.kind == CSAW_BIAS_NODE2VEC || b.kind == CSAW_BIAS_MDRW || b.kind == CSAW_BIAS_MH ||
        b.kind == CSAW_BIAS_RESTART || b.kind == CSAW_BIAS_JUMP)
        return fail(CSAW_ERR_INVALID_ARG, "node2vec / MDRW / MH / restart / jump are walk selectors (use csaw_walk)");
    if (b.kind == CSAW_BIAS_WEIGHT && !g->w)
        return fail(CSAW_ERR_INVALID_ARG, "CSAW_BIAS_WEIGHT needs a graph created with edge weights");
    if (!num_edges) return fail(CSAW_ERR_INVALID_ARG, "num_edges is NULL");
    *num_edges = 0;
    if (depth < 1 || depth > 255) return fail(CSAW_ERR_INVALID_ARG, "depth must be in [1, 255]");
    if (n < 0 || capacity < 0) return fail(CSAW_ERR_INVALID_ARG, "negative n_instances / capacity");
    if (b.kind == CSAW_BIAS_FOREST_FIRE && !(b.pf >= 0.0 && b.pf < 1.0))
        return fail(CSAW_ERR_INVALID_ARG, "forest fire needs pf in [0, 1)");
    if (b.kind != CSAW_BIAS_FOREST_FIRE && b.kind != CSAW_BIAS_SNOWBALL) {
        if (!fanout) return fail(CSAW_ERR_INVALID_ARG, "fanout is NULL");
        for (int d = 0; d < depth; ++d)
            if (fanout[d] < 0 || fanout[d] >= (1 << 14)) return fail(CSAW_ERR_INVALID_ARG, "fanout must be in [0, 2^14)");
    }
    if (instance_base + static_cast<uint64_t>(n) > 0xFFFFFFFFull)
        return fail(CSAW_ERR_INVALID_ARG, "instance ids must fit in 32 bits");
    if (g->oom && b.kind == CSAW_BIAS_LAYER && !g->oomst.zerocopy)
        return fail(CSAW_ERR_UNSUPPORTED, "OOM partition scheduling implements neighbor sampling and forest fire "
                                          "(layer pools span partitions; use CSAW_GRAPH_OOM_ZEROCOPY)");
    if (!offsets) return fail(CSAW_ERR_INVALID_ARG, "offsets is NULL");
    if (n > 0 && !seeds) return fail(CSAW_ERR_INVALID_ARG, "seeds is NULL");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (capacity > 0 && (!src || !dst || !edge_depth)) return fail(CSAW_ERR_INVALID_ARG, "src/dst/edge_depth is NULL");
    const PtrKind ks = n == 0 ? PtrKind::Device : ptr_kind(seeds, g->device);
    const PtrKind ko = ptr_kind(offsets, g->device);
    const PtrKind kd = capacity == 0 ? PtrKind::Device : ptr_kind(dst, g->device);
    if (ks == PtrKind::OtherDevice || ko == PtrKind::OtherDevice || kd == PtrKind::OtherDevice)
        return fail(CSAW_ERR_INVALID_ARG, "seeds/offsets/outputs live on another GPU than the graph");
    // src, dst and edge_depth are written by the same kernels: they must share one location class
    if (capacity > 0 && (ptr_kind(src, g->device) != kd || ptr_kind(edge_depth, g->device) != kd))
        return fail(CSAW_ERR_INVALID_ARG, "src, dst and edge_depth must all be device, all pinned or all pageable host "
                                          "buffers");
    const bool seeds_dev = ks == PtrKind::Device;
    const bool offs_dev = ko == PtrKind::Device;
    const bool out_dev = kd == PtrKind::Device;
    CallOrder order(g, st);
    const uint32_t* d_seeds = seeds;
    if (!seeds_dev) {
        void* p;
        CSAW_TRY(g->scratch.get(SL_SEEDS, sizeof(uint32_t) * n, &p));
        CSAW_CUDA(cudaMemcpyAsync(p, seeds, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st));
        d_seeds = static_cast<const uint32_t*>(p);
    }
    uint64_t* d_offs = offsets;
    if (!offs_dev) {
        void* p;
        CSAW_TRY(g->scratch.get(SL_OFFS, sizeof(uint64_t) * (n + 1), &p));
        d_offs = static_cast<uint64_t*>(p);
    }
    PinnedOut po{nullptr, nullptr, nullptr};
    if (!out_dev) {
        po.src = static_cast<uint32_t*>(pinned_device_ptr(src));
        po.dst = static_cast<uint32_t*>(pinned_device_ptr(dst));
        po.dep = static_cast<uint8_t*>(pinned_device_ptr(edge_depth));
    }
    if (!offs_dev) po.offs = static_cast<uint64_t*>(pinned_device_ptr(offsets));
    const bool any_pinned = (po.src && po.dst && po.dep) || po.offs;
    csaw_status s = run_sample(g, b, fanout, depth, d_seeds, n, instance_base, rng_seed, d_offs, src, dst,
                               edge_depth, capacity, num_edges, out_dev, st, any_pinned ? &po : nullptr);
    if (s != CSAW_OK && s != CSAW_ERR_CAPACITY) return s;
    if (!offs_dev && !po.offs_done) {
        CSAW_CUDA(cudaMemcpyAsync(offsets, d_offs, sizeof(uint64_t) * (n + 1), cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaStreamSynchronize(st));
    }
    return s;
}

// ---------------------------------------------------------------- test hooks
__global__ void k_philox(const uint4* __restrict__ ctr, uint2 key, uint4* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = philox4x32_10(ctr[i], key);
}

CSAW_API csaw_status csaw_philox(const uint32_t* ctr, const uint32_t* key, uint32_t* out, int64_t n) {
    clear_error();
    if (n <= 0) return CSAW_OK;
    if (!ctr || !key || !out) return fail(CSAW_ERR_INVALID_ARG, "NULL argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(CSAW_ERR_CUDA, "no CUDA device");
    }
    uint32_t hk[2];
    CSAW_CUDA(cudaMemcpy(hk, key, sizeof(hk), cudaMemcpyDefault));
    uint4 *dc = nullptr, *doo = nullptr;
    CSAW_CUDA(cudaMalloc(&dc, sizeof(uint4) * n));
    CSAW_CUDA(cudaMalloc(&doo, sizeof(uint4) * n));
    cudaMemcpy(dc, ctr, sizeof(uint4) * n, cudaMemcpyDefault);
    k_philox<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256>>>(dc, make_uint2(hk[0], hk[1]), doo, n);
    cudaError_t e = cudaMemcpy(out, doo, sizeof(uint4) * n, cudaMemcpyDefault);
    cudaFree(dc);
    cudaFree(doo);
    if (e != cudaSuccess) return cuda_fail(e, "csaw_philox", __FILE__, __LINE__);
    return CSAW_OK;
}

__global__ void k_selftest_curand(int64_t n, unsigned long long* mism) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = static_cast<uint32_t>(i * 2654435761ull), b = static_cast<uint32_t>(i >> 3) ^ 0x5bd1e995u;
        const uint4 c = make_uint4(a, b, a ^ 0xdeadbeefu, static_cast<uint32_t>(i));
        const uint2 k = make_uint2(b * 7u + 1u, a + 12345u);
        const uint4 mine = philox4x32_10(c, k);
        const uint4 ref = curand_Philox4x32_10(c, k);
        if (mine.x != ref.x || mine.y != ref.y || mine.z != ref.z || mine.w != ref.w) atomicAdd(mism, 1ull);
    }
}

CSAW_API csaw_status csaw_selftest_curand(int64_t n, int64_t* mismatches) {
    clear_error();
    if (!mismatches) return fail(CSAW_ERR_INVALID_ARG, "NULL argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(CSAW_ERR_CUDA, "no CUDA device");
    }
    unsigned long long* d = nullptr;
    CSAW_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
    cudaMemset(d, 0, sizeof(unsigned long long));
    k_selftest_curand<<<1024, 256>>>(n, d);
    unsigned long long h = 0;
    cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "selftest", __FILE__, __LINE__);
    *mismatches = static_cast<int64_t>(h);
    return CSAW_OK;
}

}  // extern "C"
