// oom.cu — out-of-memory mode (§5): graph partitions, workload-aware
// partition scheduling and batched multi-instance sampling under a device budget.
//
// The CSR lives in pinned host memory; the device keeps row_ptr + deg (needed by
// VERTEXBIAS / EDGEBIAS = degree for every vertex, "decide which partition a
// vertex belongs to in constant time") and R arena slots, each holding the
// col_idx slice of one partition (contiguous equal vertex range).
// One frontier queue per partition holds the instances whose next selection
// needs that partition (batched multi-instance queue).  Every wave:
//   1. count active instances per partition;
//   2. keep resident partitions that still have work, fill the free / empty
//      slots with the busiest non-resident partitions (ties -> lower id; only
//      empty-queue residents are evicted; reading R23);
//   3. cudaMemcpyAsync each new partition into its slot and launch one kernel per
//      active partition on its own stream, CTAs proportional to
//      its active count (thread-block balancing; R24);
//   4. a kernel advances each of its instances while the next pick stays in its
//      partition, then appends the instance to the owner's queue.
// Results are identical to the in-memory path: every draw is keyed by
// (instance, step), never by schedule (R7, R22).
#include <cuda_runtime.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "select.cuh"

namespace csaw {

constexpr int OOM_WARPS = 8;
constexpr int OOM_MAXP = 64;   // partitions supported by the scheduler

// Partitions whose col slice is resident and complete when a kernel starts.
struct ReadyMap {
    int32_t slot[OOM_MAXP];     // arena slot, or -1
    int64_t ebeg[OOM_MAXP];     // first CSR entry of the partition
    const uint32_t* slots;      // arena base
    int64_t slot_edges;
    __device__ __forceinline__ const uint32_t* col_of(uint32_t q) const {   // col[] view for partition q
        return slot[q] < 0 ? nullptr : slots + static_cast<int64_t>(slot[q]) * slot_edges - ebeg[q];
    }
};

struct Owner {   // equal contiguous ranges, remainder to the lowest partitions (R23)
    uint64_t base;   // V / P
    uint64_t rem;    // V % P
    __device__ __forceinline__ uint32_t operator()(uint32_t v) const {
        const uint64_t big = rem * (base + 1);
        if (v < big) return static_cast<uint32_t>(v / (base + 1));
        return static_cast<uint32_t>(rem + (v - big) / base);
    }
};

struct MdrwOom {
    // per-instance MDRW state (global memory: instances migrate between kernels)
    uint32_t* pool_v;     // [n][m]
    uint32_t* bias;       // [n][m]
    uint64_t* blk;        // [n][nblk]
    uint64_t* T;          // [n]
    uint32_t* tstep;      // [n] next step to take
    uint32_t* pend_slot;  // [n] pending pick (slot) for step tstep
    // queues: [P][n] instance ids; counts [P]
    uint32_t* qin;
    uint32_t* qout;
    uint32_t* cnt_in;
    uint32_t* cnt_out;
};

struct OomArgs {
    const int64_t* __restrict__ rp;
    const uint32_t* __restrict__ deg;
    const uint32_t* __restrict__ seeds;
    uint64_t n;
    uint32_t m, nblk;
    int32_t L;
    uint32_t ibase;
    uint2 key;
    uint32_t* __restrict__ out;   // [n][L][2]
    MdrwOom s;
    Owner own;
    uint32_t P;
};

// VERTEXBIAS = degree over the instance's pool (slot order, R18): ITS by a warp scan
// over the block totals, then over the selected block (identical to a flat scan).
__device__ __forceinline__ uint32_t mdrw_pick(const OomArgs& a, uint64_t i, uint32_t t) {
    const int lane = lane_id();
    const uint64_t T = a.s.T[i];
    const uint64_t x = below(draw_u64(a.key, a.ibase + static_cast<uint32_t>(i), t, 0u, word3(PURPOSE_VERTEX, 0, 0)), T);
    const uint64_t* blk = a.s.blk + i * a.nblk;
    uint64_t base = 0, blo = 0;
    uint32_t bsel = 0;
    for (uint32_t g0 = 0; g0 < a.nblk; g0 += 32) {
        const uint64_t vb = (g0 + lane < a.nblk) ? blk[g0 + lane] : 0;
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
    const uint32_t s0 = bsel * 32 + lane;
    const uint32_t e = s0 < a.m ? a.s.bias[i * a.m + s0] : 0u;
    const uint64_t incl2 = warp_incl_scan(static_cast<uint64_t>(e)) + blo;
    const unsigned hit2 = __ballot_sync(FULL, incl2 > x);
    return bsel * 32 + (__ffs(hit2) - 1);
}

__global__ void __launch_bounds__(OOM_WARPS * 32) k_mdrw_oom_init(OomArgs a) {
    const int lane = lane_id();
    for (uint64_t i = global_warp_id(); i < a.n; i += total_warps()) {
        uint64_t T = 0;
        for (uint32_t b = 0; b < a.nblk; ++b) {
            const uint32_t s = b * 32 + lane;
            uint32_t d = 0;
            if (s < a.m) {
                const uint32_t v = a.seeds[i * a.m + s];
                d = __ldg(a.deg + v);
                a.s.pool_v[i * a.m + s] = v;
                a.s.bias[i * a.m + s] = d;
            }
            const uint64_t tot = warp_sum(static_cast<uint64_t>(d));
            if (lane == 0) a.s.blk[i * a.nblk + b] = tot;
            T += tot;
        }
        __syncwarp();
        if (lane == 0) { a.s.T[i] = T; a.s.tstep[i] = 0; }
        __syncwarp();
        if (a.L == 0) continue;
        if (T == 0) {   // no positive-degree vertex in the pool: the walk ends (R20)
            for (uint64_t k = lane; k < static_cast<uint64_t>(a.L) * 2; k += 32) a.out[i * a.L * 2 + k] = NONE;
            continue;
        }
        const uint32_t slot = mdrw_pick(a, i, 0);
        if (lane == 0) {
            a.s.pend_slot[i] = slot;
            const uint32_t p = a.own(a.s.pool_v[i * a.m + slot]);
            const uint32_t pos = atomicAdd(a.s.cnt_in + p, 1u);
            a.s.qin[static_cast<uint64_t>(p) * a.n + pos] = static_cast<uint32_t>(i);
        }
    }
}

// One kernel per active partition p (its queue); an instance keeps stepping while
// its next pick lies in a partition that is resident and ready (rm), then joins the
// queue of the partition it needs.
__global__ void __launch_bounds__(OOM_WARPS * 32) k_mdrw_oom_part(OomArgs a, uint32_t p, ReadyMap rm,
                                                                  const uint32_t* __restrict__ qlist, uint32_t qn) {
    const int lane = lane_id();
    for (uint64_t j = global_warp_id(); j < qn; j += total_warps()) {
        const uint64_t i = qlist[j];
        const uint32_t inst = a.ibase + static_cast<uint32_t>(i);
        uint32_t t = a.s.tstep[i];
        uint32_t slot = a.s.pend_slot[i];
        uint32_t* pv = a.s.pool_v + i * a.m;
        uint32_t* bias = a.s.bias + i * a.m;
        uint64_t* blk = a.s.blk + i * a.nblk;
        uint32_t* orow = a.out + i * static_cast<uint64_t>(a.L) * 2;
        const uint32_t* colq = rm.col_of(p);
        for (;;) {
            // step t at the picked slot; its vertex v is owned by p
            if (lane == 0) {
                const uint32_t v = pv[slot];
                const uint32_t d = bias[slot];
                const int64_t rb = __ldg(a.rp + v);
                const uint64_t jj = below(draw_u64(a.key, inst, t, 0u, word3(PURPOSE_EDGE, 0, 0)), d);
                const uint32_t u = __ldg(colq + rb + jj);
                const uint32_t du = __ldg(a.deg + u);
                orow[2 * t] = v;
                orow[2 * t + 1] = u;
                pv[slot] = u;
                bias[slot] = du;
                blk[slot / 32] = blk[slot / 32] + du - d;
                a.s.T[i] = a.s.T[i] + du - d;
            }
            __syncwarp();
            ++t;
            if (t >= static_cast<uint32_t>(a.L)) break;
            slot = mdrw_pick(a, i, t);
            const uint32_t q = a.own(pv[slot]);
            colq = rm.col_of(q);
            if (colq == nullptr) {
                if (lane == 0) {
                    a.s.tstep[i] = t;
                    a.s.pend_slot[i] = slot;
                    const uint32_t pos = atomicAdd(a.s.cnt_out + q, 1u);
                    a.s.qout[static_cast<uint64_t>(q) * a.n + pos] = static_cast<uint32_t>(i);
                }
                break;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- shared scheduler pieces
std::vector<WavePick> oom_plan_wave(OomState& os, const std::vector<uint64_t>& cnt) {
    const int32_t P = os.P, R = os.R;
    std::vector<int32_t>& res = os.resident;
    std::vector<int32_t> slot_of(P, -1);
    for (int s = 0; s < R; ++s)
        if (res[s] >= 0) slot_of[res[s]] = s;
    std::vector<WavePick> w;
    std::vector<bool> used(R, false);
    if (os.ws) {
        // residents with work stay (released only when their queue is empty)
        for (int s = 0; s < R; ++s)
            if (res[s] >= 0 && cnt[res[s]] > 0) { w.push_back({res[s], s, false}); used[s] = true; }
        // free / idle slots take the busiest non-resident partitions (ties -> lower id, R23)
        std::vector<int32_t> order(P);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return cnt[x] > cnt[y]; });
        for (int32_t p : order) {
            if (static_cast<int>(w.size()) >= R || cnt[p] == 0) break;
            if (slot_of[p] >= 0) continue;
            int victim = -1;
            for (int s = 0; s < R && victim < 0; ++s)
                if (!used[s]) victim = s;
            if (victim < 0) break;
            if (res[victim] >= 0) slot_of[res[victim]] = -1;
            res[victim] = p;
            slot_of[p] = victim;
            used[victim] = true;
            w.push_back({p, victim, true});
        }
        return w;
    }
    // ablation (no WS): next R non-empty partitions in cyclic id order, FIFO eviction
    std::vector<int32_t> picks;
    int32_t last = -1;
    for (int32_t k = 0; k < P && static_cast<int>(picks.size()) < R; ++k) {
        const int32_t p = (os.rr + k) % P;
        if (cnt[p] > 0) { picks.push_back(p); last = p; }
    }
    if (last >= 0) os.rr = (last + 1) % P;
    for (int32_t p : picks)
        if (slot_of[p] >= 0) { w.push_back({p, slot_of[p], false}); used[slot_of[p]] = true; }
    for (int32_t p : picks) {
        if (slot_of[p] >= 0) continue;
        int victim = -1;
        for (int k = 0; k < R && victim < 0; ++k) {
            const int s = (os.fifo + k) % R;
            if (!used[s]) victim = s;
        }
        if (victim < 0) break;
        os.fifo = (victim + 1) % R;
        if (res[victim] >= 0) slot_of[res[victim]] = -1;
        res[victim] = p;
        slot_of[p] = victim;
        used[victim] = true;
        w.push_back({p, victim, true});
    }
    return w;
}

csaw_status oom_load(const csaw_graph* g, int32_t p, int32_t slot, cudaEvent_t after, std::vector<cudaEvent_t>& tev) {
    auto& os = const_cast<csaw_graph*>(g)->oomst;
    cudaStream_t ss = os.streams[slot % os.S];
    cudaEvent_t t0, t1;
    CSAW_CUDA(cudaEventCreate(&t0));
    CSAW_CUDA(cudaEventCreate(&t1));
    CSAW_CUDA(cudaStreamWaitEvent(ss, after, 0));
    CSAW_CUDA(cudaEventRecord(t0, ss));
    const int64_t ne = os.ebeg[p + 1] - os.ebeg[p];
    // host -> device (the paper's §5 store) or peer HBM -> local HBM over NVLink (NEXT-4(i))
    CSAW_CUDA(cudaMemcpyAsync(os.d_slots + static_cast<int64_t>(slot) * os.slot_edges, os.src_col + os.ebeg[p],
                              sizeof(uint32_t) * ne, cudaMemcpyDefault, ss));
    CSAW_CUDA(cudaEventRecord(t1, ss));
    tev.push_back(t0);
    tev.push_back(t1);
    g->stats.partition_loads += 1;
    g->stats.h2d_bytes += sizeof(uint32_t) * ne;
    return CSAW_OK;
}

void oom_account_transfers(const csaw_graph* g, std::vector<cudaEvent_t>& tev) {
    double tms = 0;
    for (size_t k = 0; k + 1 < tev.size(); k += 2) {
        float ms = 0;
        cudaEventSynchronize(tev[k + 1]);
        cudaEventElapsedTime(&ms, tev[k], tev[k + 1]);
        tms += ms;
        cudaEventDestroy(tev[k]);
        cudaEventDestroy(tev[k + 1]);
    }
    tev.clear();
    g->stats.transfer_ms += tms;
}

int oom_blocks(const OomState& os, int blocks_total, uint64_t c, uint64_t wave_total, size_t nchosen, int warps) {
    uint64_t b = os.bal ? blocks_total * c / std::max<uint64_t>(wave_total, 1)            // P:850, R24
                        : static_cast<uint64_t>(blocks_total) / std::max<size_t>(nchosen, 1);
    b = std::max<uint64_t>(b, 1);
    if (os.bal) b = std::min<uint64_t>(b, (c + warps - 1) / warps);   // no idle CTAs
    return static_cast<int>(b);
}

// Wave loop shared by the walk-style OOM workloads (MDRW, degree / uniform walks):
// every wave plans the partitions, loads the fresh ones, launches one kernel per
// partition on the slot's stream (ready map = residents not being overwritten +
// the partition itself), then merges the per-partition out-queues.
template <class Launch>
static csaw_status oom_walk_waves(const csaw_graph* g, uint64_t n, uint32_t* qin, uint32_t* qout, uint32_t* cnt_in,
                                  uint32_t* cnt_out, int warps, cudaStream_t st, Launch&& launch) {
    auto& os = const_cast<csaw_graph*>(g)->oomst;
    const uint32_t P = static_cast<uint32_t>(os.P);
    void* hmb;
    CSAW_TRY(g->pinned.get(4096, &hmb));
    uint32_t* hcnt = static_cast<uint32_t*>(hmb);   // [0,P) in, [P,2P) out
    const int blocks_total = g->num_sms * 8;
    cudaEvent_t evs;
    CSAW_CUDA(cudaEventCreateWithFlags(&evs, cudaEventDisableTiming));
    std::vector<cudaEvent_t> tev;
    std::vector<uint64_t> in_cnt(P), out_cnt(P);
    for (;;) {
        CSAW_CUDA(cudaMemcpyAsync(hcnt, cnt_in, P * 4, cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaStreamSynchronize(st));
        uint64_t active_total = 0;
        for (uint32_t p = 0; p < P; ++p) { in_cnt[p] = hcnt[p]; active_total += in_cnt[p]; }
        if (active_total == 0) break;
        const std::vector<WavePick> wave = oom_plan_wave(os, in_cnt);
        CSAW_CUDA(cudaEventRecord(evs, st));
        for (const WavePick& w : wave)
            if (w.fresh) CSAW_TRY(oom_load(g, w.p, w.slot, evs, tev));
        ReadyMap rm;
        rm.slots = os.d_slots;
        rm.slot_edges = os.slot_edges;
        for (int q = 0; q < OOM_MAXP; ++q) { rm.slot[q] = -1; rm.ebeg[q] = 0; }
        for (uint32_t q = 0; q < P; ++q) rm.ebeg[q] = os.ebeg[q];
        for (const WavePick& w : wave)
            if (!w.fresh) rm.slot[w.p] = w.slot;
        for (int s = 0; s < os.R; ++s) {   // idle residents not overwritten this wave are ready too
            bool in_wave = false;
            for (const WavePick& w : wave) in_wave |= w.slot == s;
            if (!in_wave && os.resident[s] >= 0) rm.slot[os.resident[s]] = s;
        }
        uint64_t wave_total = 0;
        for (const WavePick& w : wave) wave_total += in_cnt[w.p];
        for (const WavePick& w : wave) {
            cudaStream_t ss = os.streams[w.slot % os.S];
            CSAW_CUDA(cudaStreamWaitEvent(ss, evs, 0));
            const int blocks = oom_blocks(os, blocks_total, in_cnt[w.p], wave_total, wave.size(), warps);
            ReadyMap rmp = rm;
            rmp.slot[w.p] = w.slot;
            CSAW_TRY(hot_begin(g, ss));
            launch(static_cast<uint32_t>(w.p), rmp, qin + static_cast<uint64_t>(w.p) * n,
                   static_cast<uint32_t>(in_cnt[w.p]), blocks, ss);
            note_launch();
            CSAW_CUDA(cudaGetLastError());
            CSAW_TRY(hot_end(g, ss));
        }
        for (int s = 0; s < os.S; ++s) {
            CSAW_CUDA(cudaEventRecord(evs, os.streams[s]));
            CSAW_CUDA(cudaStreamWaitEvent(st, evs, 0));
        }
        // merge queues: sampled partitions take their out-queue; others append it
        CSAW_CUDA(cudaMemcpyAsync(hcnt + P, cnt_out, P * 4, cudaMemcpyDeviceToHost, st));
        CSAW_CUDA(cudaStreamSynchronize(st));
        for (uint32_t p = 0; p < P; ++p) {
            out_cnt[p] = hcnt[P + p];
            bool was = false;
            for (const WavePick& w : wave) was |= w.p == static_cast<int32_t>(p);
            const uint64_t keep = was ? 0 : in_cnt[p];
            if (out_cnt[p])
                CSAW_CUDA(cudaMemcpyAsync(qin + static_cast<uint64_t>(p) * n + keep, qout + static_cast<uint64_t>(p) * n,
                                          sizeof(uint32_t) * out_cnt[p], cudaMemcpyDeviceToDevice, st));
            hcnt[p] = static_cast<uint32_t>(keep + out_cnt[p]);
        }
        CSAW_CUDA(cudaMemcpyAsync(cnt_in, hcnt, P * 4, cudaMemcpyHostToDevice, st));
        CSAW_CUDA(cudaMemsetAsync(cnt_out, 0, P * 4, st));
    }
    CSAW_CUDA(cudaStreamSynchronize(st));
    oom_account_transfers(g, tev);
    cudaEventDestroy(evs);
    return CSAW_OK;
}

csaw_status run_mdrw_oom(const csaw_graph* g, const csaw_bias& b, int32_t length, const uint32_t* d_seeds, int64_t n_i,
                         uint64_t base, uint64_t seed, uint32_t* d_path, cudaStream_t st) {
    if (b.kind != CSAW_BIAS_MDRW) return fail(CSAW_ERR_UNSUPPORTED, "OOM mode implements MDRW walks (config 5)");
    const uint64_t n = static_cast<uint64_t>(n_i);
    auto& os = const_cast<csaw_graph*>(g)->oomst;
    const uint32_t m = static_cast<uint32_t>(b.pool_size);
    const uint32_t nblk = (m + 31) / 32;
    const uint32_t P = static_cast<uint32_t>(os.P);
    // device scratch (counted against the budget)
    if (P > static_cast<uint32_t>(OOM_MAXP)) return fail(CSAW_ERR_UNSUPPORTED, "OOM mode supports at most 64 partitions");
    const size_t need = n * m * 8 + n * nblk * 8 + n * 16 + 2 * static_cast<size_t>(P) * n * 4 + 2 * P * 4 + 16 * 16;
    const int64_t resident = sizeof(int64_t) * (g->V + 1) + sizeof(uint32_t) * g->V +
                             static_cast<int64_t>(os.R) * os.slot_edges * 4;
    if (resident + static_cast<int64_t>(need) > os.budget)
        return fail(CSAW_ERR_NO_MEMORY, "OOM mode: instance state (" + std::to_string(need) +
                                            " B) does not fit the device budget next to the resident graph");
    void* p0;
    CSAW_TRY(g->scratch.get(SL_TMP0, need, &p0));
    char* cur = static_cast<char*>(p0);
    auto take = [&](size_t bytes) { char* r = cur; cur += (bytes + 15) / 16 * 16; return static_cast<void*>(r); };
    OomArgs a;
    a.rp = g->row_ptr; a.deg = g->deg; a.seeds = d_seeds; a.n = n; a.m = m; a.nblk = nblk; a.L = length;
    a.ibase = static_cast<uint32_t>(base);
    a.key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    a.out = d_path;
    a.s.pool_v = static_cast<uint32_t*>(take(n * m * 4));
    a.s.bias = static_cast<uint32_t*>(take(n * m * 4));
    a.s.blk = static_cast<uint64_t*>(take(n * nblk * 8));
    a.s.T = static_cast<uint64_t*>(take(n * 8));
    a.s.tstep = static_cast<uint32_t*>(take(n * 4));
    a.s.pend_slot = static_cast<uint32_t*>(take(n * 4));
    a.s.qin = static_cast<uint32_t*>(take(static_cast<size_t>(P) * n * 4));
    a.s.qout = static_cast<uint32_t*>(take(static_cast<size_t>(P) * n * 4));
    a.s.cnt_in = static_cast<uint32_t*>(take(P * 4));
    a.s.cnt_out = static_cast<uint32_t*>(take(P * 4));
    a.own.base = static_cast<uint64_t>(g->V) / P;
    a.own.rem = static_cast<uint64_t>(g->V) % P;
    a.P = P;

    CSAW_CUDA(cudaMemsetAsync(a.s.cnt_in, 0, P * 4, st));
    CSAW_CUDA(cudaMemsetAsync(a.s.cnt_out, 0, P * 4, st));
    CSAW_TRY(stats_begin(g, st));
    const int blocks_total = g->num_sms * 8;
    if (n > 0) {
        k_mdrw_oom_init<<<std::max(1, (int)std::min<uint64_t>((n + OOM_WARPS - 1) / OOM_WARPS, blocks_total)),
                          OOM_WARPS * 32, 0, st>>>(a);
        note_launch();
        CSAW_CUDA(cudaGetLastError());
    }
    CSAW_TRY(oom_walk_waves(g, n, a.s.qin, a.s.qout, a.s.cnt_in, a.s.cnt_out, OOM_WARPS, st,
                            [&](uint32_t p, const ReadyMap& rm, const uint32_t* ql, uint32_t qn, int blocks,
                                cudaStream_t ss) {
                                k_mdrw_oom_part<<<blocks, OOM_WARPS * 32, 0, ss>>>(a, p, rm, ql, qn);
                            }));
    CSAW_TRY(stats_end(g, st));
    g->stats.sampled_edges = n * static_cast<uint64_t>(length);
    g->stats.pools = n * static_cast<uint64_t>(length);
    return CSAW_OK;
}

// ---------------------------------------------------------------- degree / uniform walks (Fig. 13(b))
// Walker state in global memory (walkers migrate between partition kernels):
// current vertex and next step.  A walker keeps stepping while its current
// vertex's partition is ready; the path is written step by step.
struct WalkOomArgs {
    const int64_t* __restrict__ rp;
    const uint32_t* __restrict__ deg;
    uint64_t n;
    int32_t L;
    uint32_t ibase;
    uint2 key;
    uint32_t* __restrict__ path;     // [n][L+1]
    uint32_t* cur;                   // [n]
    uint32_t* tstep;                 // [n]
    uint32_t* qin;
    uint32_t* qout;
    uint32_t* cnt_in;
    uint32_t* cnt_out;
    unsigned long long* counters;    // [0] scanned, [1] steps
    Owner own;
    const uint64_t* ccache;          // chunk-total cache (degree pools), optional
};

__global__ void __launch_bounds__(OOM_WARPS * 32) k_walk_oom_init(WalkOomArgs a, const uint32_t* __restrict__ seeds) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = seeds[i];
        uint32_t* row = a.path + i * (static_cast<uint64_t>(a.L) + 1);
        row[0] = s;
        a.cur[i] = s;
        a.tstep[i] = 0;
        if (a.L == 0) continue;
        if (__ldg(a.deg + s) == 0) {   // R20: the walk ends, padded with NONE
            for (int32_t t = 1; t <= a.L; ++t) row[t] = NONE;
            continue;
        }
        const uint32_t p = a.own(s);
        const uint32_t pos = atomicAdd(a.cnt_in + p, 1u);
        a.qin[static_cast<uint64_t>(p) * a.n + pos] = static_cast<uint32_t>(i);
    }
}

template <bool kUniform>
__global__ void __launch_bounds__(OOM_WARPS * 32) k_walk_oom_part(WalkOomArgs a, uint32_t p, ReadyMap rm,
                                                                  const uint32_t* __restrict__ qlist, uint32_t qn) {
    __shared__ uint64_t tab_all[OOM_WARPS][TAB];
    uint64_t* tab = tab_all[threadIdx.x >> 5];
    const int lane = lane_id();
    unsigned long long scanned = 0, steps = 0;
    for (uint64_t j = global_warp_id(); j < qn; j += total_warps()) {
        const uint64_t i = qlist[j];
        const uint32_t inst = a.ibase + static_cast<uint32_t>(i);
        uint32_t t = a.tstep[i];
        uint32_t v = a.cur[i];
        uint32_t* row = a.path + i * (static_cast<uint64_t>(a.L) + 1);
        const uint32_t* colq = rm.col_of(p);
        for (;;) {
            const int64_t b0 = __ldg(a.rp + v);
            const uint32_t d = static_cast<uint32_t>(__ldg(a.rp + v + 1) - b0);   // > 0 (checked on entry)
            const uint64_t U = draw_u64(a.key, inst, t, 0u, word3(PURPOSE_EDGE, 0, 0));
            uint32_t nxt;
            if constexpr (kUniform) {
                nxt = __ldg(colq + b0 + below(U, d));
            } else {
                DegreePool P{colq, a.deg, static_cast<uint64_t>(b0), d, a.ccache};
                const Ctps C = build_ctps(P, tab);
                nxt = select_wr(P, C, tab, U);
                scanned += (a.ccache && C.m) ? 32u * C.m : d;
            }
            ++steps;
            ++t;
            if (lane == 0) row[t] = nxt;
            if (t >= static_cast<uint32_t>(a.L)) break;
            if (nxt == NONE || __ldg(a.deg + nxt) == 0) {   // R20: pad the rest
                for (uint32_t r = t + 1 + lane; r <= static_cast<uint32_t>(a.L); r += 32) row[r] = NONE;
                break;
            }
            v = nxt;
            const uint32_t q = a.own(v);
            colq = rm.col_of(q);
            if (colq == nullptr) {
                if (lane == 0) {
                    a.tstep[i] = t;
                    a.cur[i] = v;
                    const uint32_t pos = atomicAdd(a.cnt_out + q, 1u);
                    a.qout[static_cast<uint64_t>(q) * a.n + pos] = static_cast<uint32_t>(i);
                }
                break;
            }
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (scanned) atomicAdd(a.counters + 0, scanned);
        if (steps) atomicAdd(a.counters + 1, steps);
    }
}

csaw_status run_walk_oom(const csaw_graph* g, const csaw_bias& b, int32_t length, const uint32_t* d_seeds, int64_t n_i,
                         uint64_t base, uint64_t seed, uint32_t* d_path, cudaStream_t st) {
    if (b.kind != CSAW_BIAS_DEGREE && b.kind != CSAW_BIAS_UNIFORM)
        return fail(CSAW_ERR_UNSUPPORTED, "OOM partition mode implements MDRW, degree and uniform walks");
    const uint64_t n = static_cast<uint64_t>(n_i);
    auto& os = const_cast<csaw_graph*>(g)->oomst;
    const uint32_t P = static_cast<uint32_t>(os.P);
    if (P > static_cast<uint32_t>(OOM_MAXP)) return fail(CSAW_ERR_UNSUPPORTED, "OOM mode supports at most 64 partitions");
    const size_t need = n * 8 + 2 * static_cast<size_t>(P) * n * 4 + 2 * P * 4 + 64 + 16 * 16;
    const int64_t resident = sizeof(int64_t) * (g->V + 1) + sizeof(uint32_t) * g->V +
                             static_cast<int64_t>(os.R) * os.slot_edges * 4;
    if (resident + static_cast<int64_t>(need) > os.budget)
        return fail(CSAW_ERR_NO_MEMORY, "OOM mode: walker state (" + std::to_string(need) +
                                            " B) does not fit the device budget next to the resident graph");
    void* p0;
    CSAW_TRY(g->scratch.get(SL_TMP0, need, &p0));
    char* curp = static_cast<char*>(p0);
    auto take = [&](size_t bytes) { char* r = curp; curp += (bytes + 15) / 16 * 16; return static_cast<void*>(r); };
    WalkOomArgs a;
    a.ccache = g->ccache;
    a.rp = g->row_ptr; a.deg = g->deg; a.n = n; a.L = length; a.ibase = static_cast<uint32_t>(base);
    a.key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    a.path = d_path;
    a.cur = static_cast<uint32_t*>(take(n * 4));
    a.tstep = static_cast<uint32_t*>(take(n * 4));
    a.qin = static_cast<uint32_t*>(take(static_cast<size_t>(P) * n * 4));
    a.qout = static_cast<uint32_t*>(take(static_cast<size_t>(P) * n * 4));
    a.cnt_in = static_cast<uint32_t*>(take(P * 4));
    a.cnt_out = static_cast<uint32_t*>(take(P * 4));
    a.counters = static_cast<unsigned long long*>(take(64));
    a.own.base = static_cast<uint64_t>(g->V) / P;
    a.own.rem = static_cast<uint64_t>(g->V) % P;
    CSAW_CUDA(cudaMemsetAsync(a.cnt_in, 0, P * 4, st));
    CSAW_CUDA(cudaMemsetAsync(a.cnt_out, 0, P * 4, st));
    CSAW_CUDA(cudaMemsetAsync(a.counters, 0, 64, st));
    CSAW_TRY(stats_begin(g, st));
    if (n > 0) {
        const int ib = static_cast<int>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(g->num_sms) * 8));
        k_walk_oom_init<<<ib, OOM_WARPS * 32, 0, st>>>(a, d_seeds);
        note_launch();
        CSAW_CUDA(cudaGetLastError());
    }
    const bool uni = b.kind == CSAW_BIAS_UNIFORM;
    CSAW_TRY(oom_walk_waves(g, n, a.qin, a.qout, a.cnt_in, a.cnt_out, OOM_WARPS, st,
                            [&](uint32_t p, const ReadyMap& rm, const uint32_t* ql, uint32_t qn, int blocks,
                                cudaStream_t ss) {
                                if (uni) k_walk_oom_part<true><<<blocks, OOM_WARPS * 32, 0, ss>>>(a, p, rm, ql, qn);
                                else k_walk_oom_part<false><<<blocks, OOM_WARPS * 32, 0, ss>>>(a, p, rm, ql, qn);
                            }));
    CSAW_TRY(stats_end(g, st));
    unsigned long long hc[2] = {0, 0};
    CSAW_CUDA(cudaMemcpyAsync(hc, a.counters, sizeof(hc), cudaMemcpyDeviceToHost, st));
    CSAW_CUDA(cudaStreamSynchronize(st));
    g->stats.neighbours_scanned = hc[0];
    g->stats.pools = hc[1];
    g->stats.sampled_edges = n * static_cast<uint64_t>(length);
    return CSAW_OK;
}

}  // namespace csaw
