// internal.h — host runtime shared by the C ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/csaw.h"

namespace csaw {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
void clear_error();

struct Status {
    csaw_status code;
    Status(csaw_status c = CSAW_OK) : code(c) {}
    bool ok() const { return code == CSAW_OK; }
};

csaw_status cuda_fail(cudaError_t e, const char* what, const char* file, int line);

// zero padding after per-edge arrays read as 16 B vectors (vscan.cuh: one warp row = 128 entries)
#define VSCAN_PAD 128
// node2vec index records (n2v_index.cu): N2X_P inline member positions / splitters after a
// 32 B header; 24 -> 128 B records (one DRAM line, what a 64 B random read moves anyway)
#ifndef N2X_P
#define N2X_P 24
#endif
constexpr int N2X_U4 = 2 + N2X_P / 4;   // record size in uint4

#define CSAW_CUDA(call)                                                         \
    do {                                                                        \
        cudaError_t e_ = (call);                                                \
        if (e_ != cudaSuccess) return ::csaw::cuda_fail(e_, #call, __FILE__, __LINE__); \
    } while (0)

#define CSAW_TRY(expr)                                                          \
    do {                                                                        \
        csaw_status s_ = (expr);                                                \
        if (s_ != CSAW_OK) return s_;                                           \
    } while (0)

inline csaw_status fail(csaw_status s, const std::string& msg) {
    set_error(msg);
    return s;
}

// ---------------------------------------------------------------- device scratch
// Named growable device buffers owned by a graph, reused across calls.  Growth
// frees + re-allocates (stream-ordered alloc is avoided to keep the memory
// footprint predictable under an OOM budget).
class Scratch {
public:
    ~Scratch();
    // Returns a device buffer of at least `bytes` for slot `slot`.
    csaw_status get(int slot, size_t bytes, void** out);
    size_t bytes_held() const;
    void release_all();
private:
    struct Buf { void* p = nullptr; size_t n = 0; };
    std::vector<Buf> bufs_;
};

// A pinned host staging buffer (for host-pointer arguments).
class PinnedBuf {
public:
    ~PinnedBuf();
    csaw_status get(size_t bytes, void** out);
private:
    void* p_ = nullptr;
    size_t n_ = 0;
};

// ---------------------------------------------------------------- out-of-memory state
struct OomState {
    int32_t P = 0;                 // partitions
    int32_t R = 0;                 // resident slots
    int32_t S = 0;                 // streams
    int64_t budget = 0;
    bool zerocopy = false;         // CSAW_GRAPH_OOM_ZEROCOPY: kernels read h_col in place
    bool want_ccache = false;      // the chunk-total cache fits the budget (built after validation)
    std::vector<int64_t> bounds;   // vertex bounds [P+1]
    std::vector<int64_t> ebeg;     // first edge of partition p
    int64_t slot_edges = 0;        // capacity of an arena slot in col entries
    uint32_t* h_col = nullptr;     // pinned host col_idx (full graph), unless the store is a peer GPU's
    uint32_t* d_store = nullptr;   // CSAW_GRAPH_OOM_PEER_STORE: col_idx in store_device's HBM
    int store_device = -1;
    const uint32_t* src_col = nullptr;   // the partition store: h_col or d_store (UVA pointer)
    int64_t* h_row = nullptr;      // pinned host row_ptr
    uint32_t* d_slots = nullptr;   // R arena slots of col entries
    // zero-copy mode: col_idx[0, colc_n) resident on the device (the budget left after
    // row_ptr + deg + a run-state reserve), the rest read in place from h_col
    uint32_t* d_colc = nullptr;
    int64_t colc_n = 0;
    std::vector<int32_t> resident; // partition id per slot (-1 = empty)
    std::vector<cudaStream_t> streams;
    // ablation switches (Fig. 13-15): workload-aware scheduling, thread-block balancing
    bool ws = true;
    bool bal = true;
    int32_t rr = 0;                // round-robin cursor (ws off)
    int32_t fifo = 0;              // eviction cursor (ws off)
};

// One partition sampled in a wave: its arena slot and whether it is transferred now.
struct WavePick {
    int32_t p;
    int32_t slot;
    bool fresh;
};
// Choose this wave's partitions and slots from the per-partition active counts
// (updates os.resident); see oom.cu.
std::vector<WavePick> oom_plan_wave(OomState& os, const std::vector<uint64_t>& cnt);
// Enqueue the col-slice transfer of partition p into `slot` on the slot's stream,
// ordered after `after`; appends a timing event pair to tev and counts the load.
csaw_status oom_load(const csaw_graph* g, int32_t p, int32_t slot, cudaEvent_t after, std::vector<cudaEvent_t>& tev);
// Sum the transfer event pairs into stats.transfer_ms (after a sync) and destroy them.
void oom_account_transfers(const csaw_graph* g, std::vector<cudaEvent_t>& tev);
// CTAs for a partition kernel: proportional to its active count (BAL) or an even split.
int oom_blocks(const OomState& os, int blocks_total, uint64_t c, uint64_t wave_total, size_t nchosen, int warps);

}  // namespace csaw

struct csaw_graph {
    int device = 0;
    int64_t V = 0, E = 0;
    int64_t* row_ptr = nullptr;   // device [V+1] (in OOM mode: full row_ptr stays resident)
    uint32_t* col = nullptr;      // device [E] (nullptr in OOM mode)
    uint32_t* deg = nullptr;      // device [V]
    int64_t max_deg = 0;
    int64_t nonisolated = 0;
    int32_t rows_sorted = 0;
    uint64_t* cps = nullptr;      // static-bias CTPS cache [E] (CSAW_GRAPH_CTPS_CACHE), inclusive per row
    uint32_t* npos = nullptr;     // [V] positive-bias neighbours per row (cache builds only)
    uint64_t* bt = nullptr;       // fanout-32 B-tree index levels over cps (rows with d > 32)
    uint64_t* bt_off = nullptr;   // [V] start of a row's index segment in bt (= row_ptr/16 + 8 v)
    uint64_t* nmp = nullptr;      // [E] next-vertex metadata row_ptr[u] << 24 | deg(u) (walks)
    uint4* nrec = nullptr;        // [E] next-vertex record {u, deg(u), row_ptr[u] lo, hi} (MDRW)
    uint4* gbk = nullptr;         // bucketed walk index: [buckets][8] entries {S, u | k_u << 27, bucket of u, T_u}
    uint4* gmeta = nullptr;       // [V] {first bucket, k, T, 0}
    uint64_t gb_buckets = 0;
    // the same for edge weights (fp64 CTPS, float path R28): buckets of 5 SoA entries
    // {S f64[5], T_u f64[5], u | (k_u + 24) << 27 [5], bucket of u [5]}, meta {bucket, k + 24, T lo, T hi}
    uint8_t* gbw = nullptr;
    uint4* gwmeta = nullptr;
    double* cpsw = nullptr;       // [E] inclusive left-to-right fp64 prefix of the weights per row
    uint64_t gbw_buckets = 0;
    // narrow walk index (wix.cuh): built with the cache when every row total T < 2^32
    uint32_t* c32 = nullptr;      // padded leaves: S_{i+1} as u32 (wix.cuh leaf_pos)
    uint32_t* wcol = nullptr;     // padded leaves: col copy
    uint4* wrec = nullptr;        // [V] {leaf position, degree, index offset, T}
    uint32_t* whead = nullptr;    // [V][128] vertex heads (wix.cuh): record + top level / inline leaf
    uint32_t* winn = nullptr;     // internal levels (fanout 128), top level first per row
    uint64_t winn_entries = 0;    // size of winn (the records wrec follow it in the same allocation)
    uint64_t wleaf_entries = 0;   // size of c32 / wcol
    uint64_t* ccache = nullptr;   // chunk-total cache of the degree bias (select.cuh; rows of d > TAB)
    uint64_t ccache_entries = 0;
    uint32_t* tri = nullptr;      // [E] node2vec: |N(v) ∩ N(u)| per entry (symmetric sorted graphs, cache builds)
    // node2vec per-edge intersection index (n2v_index.cu, CSAW_GRAPH_N2V_INDEX)
    uint4* n2x_rec = nullptr;     // [N2X_U4 E] {offset lo, offset hi 8 | C << 8, ppos, mb}, {v, row lo, row hi 8 | deg << 8, 0}, P[N2X_P]
    uint32_t* n2x_idx = nullptr;  // member positions, n2x_total entries
    uint64_t n2x_total = 0;
    uint32_t flags = 0;           // csaw_graph_opts.flags (variant selectors are read from here)
    float* w = nullptr;           // [E + VSCAN_PAD] caller edge weights (EdgeBias = w(e), vscan.cuh), zero-padded
    uint32_t* ebias = nullptr;    // [E + VSCAN_PAD] materialised degree bias deg(col[e]) (CSAW_GRAPH_EDGE_BIAS)
    int wix_group = 8;            // lanes per walker in k_walk_wixg (32 = k_walk_wix, one warp per walker)
    int wix_leaf = 0;             // leaf fanout 32 / 64 / 128 (0 = not built)
    double cache_build_ms = 0.0;
    int num_sms = 148;
    bool oom = false;
    csaw::OomState oomst;
    mutable csaw::Scratch scratch;
    mutable csaw::PinnedBuf pinned;
    mutable csaw_run_stats stats{};
    mutable cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // completion of the previous call's work on its stream: every call's stream waits on
    // it first, so calls on different streams never overlap on the shared scratch
    mutable cudaEvent_t ev_done = nullptr;
    // pinned host walk outputs of the node2vec index kernel: chunks are copied back on this
    // stream while the next chunk walks (created on first use)
    mutable cudaStream_t copy_st = nullptr;
    mutable cudaEvent_t copy_ev[9] = {};
    // hot-kernel timing: event pairs recorded around each selection-kernel launch
    mutable std::vector<cudaEvent_t> hot_ev;
    mutable int hot_used = 0;
    // device counters still to be folded into `stats` ([0] scanned, [1] pools/steps)
    mutable const unsigned long long* pending_counters = nullptr;
    // testing / ablation: always use the level-synchronous batched sampling driver
    bool force_batched = false;
};

namespace csaw {
// scratch slot ids
enum Slot : int {
    SL_SEEDS = 0, SL_OUT, SL_OFFS, SL_SRC, SL_DST, SL_DEP, SL_COUNTS, SL_GLIST, SL_TMP0, SL_TMP1, SL_TMP2,
    SL_LEVEL_BASE = 16,          // per-level arrays: SL_LEVEL_BASE + level * 16 + k
    SL_MAX = 16 + 256 * 16
};

// Where a caller buffer lives: device memory of the graph's GPU, of another GPU (an
// error: kernels on g->device cannot dereference it without peer access), pinned
// (page-locked, device-mapped) host memory, or pageable host memory.
enum class PtrKind { Device, OtherDevice, Pinned, Pageable };
PtrKind ptr_kind(const void* p, int device);
bool is_device_ptr(const void* p, int device);
csaw_status begin_call(const csaw_graph* g);
// Orders a call after the previous one on the same graph (any stream) and records the
// call's completion on its stream when the guard goes out of scope.
struct CallOrder {
    const csaw_graph* g;
    cudaStream_t st;
    CallOrder(const csaw_graph* g_, cudaStream_t st_);
    ~CallOrder();
};

// kernels launched by the current call (per host thread)
extern thread_local uint64_t tl_launches;
inline void note_launch(uint64_t k = 1) { tl_launches += k; }
// start a call's statistics: resets counters, records ev0 on st
csaw_status stats_begin(const csaw_graph* g, cudaStream_t st);
// bracket one hot-kernel launch with events
csaw_status hot_begin(const csaw_graph* g, cudaStream_t st);
csaw_status hot_end(const csaw_graph* g, cudaStream_t st);
// end a call: records ev1, stores the launch count
csaw_status stats_end(const csaw_graph* g, cudaStream_t st);

// n2v_index.cu
csaw_status build_n2v_index(csaw_graph* g, int blocks);
csaw_status launch_node2vec_index(const csaw_graph* g, const uint32_t* seeds, uint64_t n, int32_t L, uint32_t base,
                                  uint2 key, uint32_t* path, unsigned long long* counters, uint32_t wp, uint32_t w1,
                                  uint32_t wq, cudaStream_t st);

// vwalk.cu: walks over a per-edge bias stream (weights = true: g->w, else g->ebias); group =
// warps per walker (0 = automatic; results do not depend on it)
csaw_status launch_walk_vscan(const csaw_graph* g, bool weights, const uint32_t* seeds, uint64_t n, int32_t L,
                              uint32_t base, uint2 key, uint32_t* path, unsigned long long* counters, int group,
                              cudaStream_t st);

// walk.cu / sample.cu entry points
// false if run_walk's kernel for b writes the path with scattered per-thread stores (the
// node2vec index kernel): a pinned host path is then staged in device memory and copied
bool walk_path_direct_ok(const csaw_graph* g, const csaw_bias& b);
// h_path (pinned host, optional): run_walk copies the path there itself -- the node2vec index
// walk in chunks of walkers whose copies overlap the next chunk's walk (the caller then skips
// its own copy); h_path is ignored (false returned in *copied) for every other kernel
csaw_status run_walk(const csaw_graph* g, const csaw_bias& b, int32_t length, const uint32_t* d_seeds,
                     int64_t n, uint64_t base, uint64_t seed, uint32_t* d_path, cudaStream_t st,
                     uint32_t* h_path = nullptr, bool* copied = nullptr);
// pinned host outputs, device-mapped (the fused sampler writes them directly; the batched
// driver's scattered writes stage through device scratch instead)
struct PinnedOut {
    uint32_t* src;
    uint32_t* dst;
    uint8_t* dep;
    uint64_t* offs = nullptr;     // pinned host offsets (device-mapped), or nullptr
    bool offs_done = false;       // set when the fused sampler wrote them directly
};
csaw_status run_sample(const csaw_graph* g, const csaw_bias& b, const int32_t* fanout, int32_t depth,
                       const uint32_t* d_seeds, int64_t n, uint64_t base, uint64_t seed, uint64_t* d_offsets,
                       uint32_t* src, uint32_t* dst, uint8_t* dep, int64_t capacity, int64_t* num_edges,
                       bool out_on_device, cudaStream_t st, PinnedOut* pinned = nullptr);
csaw_status run_sample_levels(const csaw_graph* g, const csaw_bias& b, const int32_t* fanout, int32_t depth,
                              const uint32_t* d_seeds, int64_t n, uint64_t base, uint64_t seed, uint64_t* d_offsets,
                              uint32_t* src, uint32_t* dst, uint8_t* dep, int64_t capacity, int64_t* num_edges,
                              bool out_on_device, cudaStream_t st);
csaw_status run_mdrw_oom(const csaw_graph* g, const csaw_bias& b, int32_t length, const uint32_t* d_seeds,
                         int64_t n, uint64_t base, uint64_t seed, uint32_t* d_path, cudaStream_t st);
csaw_status run_walk_oom(const csaw_graph* g, const csaw_bias& b, int32_t length, const uint32_t* d_seeds,
                         int64_t n, uint64_t base, uint64_t seed, uint32_t* d_path, cudaStream_t st);
}  // namespace csaw
