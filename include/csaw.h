/*
 * csaw.h — C ABI of the B200-native C-SAW hot path (arXiv 2009.09103).
 *
 * "P:n" cites line n of the paper's LaTeX; "R<n>" cites reading n
 * in DESIGN.md §3 (where the paper is silent or garbled).
 *
 * The library implements the paper's data-parallel hot path -- bias-based
 * vertex selection (§2.2, §4) inside the sampling / random-walk main loop
 * (Fig. 2(b)) -- as hand-written sm_100a CUDA kernels.  There is no
 * CPU fallback: every entry point that computes needs a CUDA device and fails
 * with CSAW_ERR_CUDA otherwise.
 *
 * Conventions shared by all entry points
 *  - Pointers are plain host or device pointers; the library detects which with
 *    cudaPointerGetAttributes.  Device pointers must live on the graph's device.
 *    Host pointers are staged through library-owned device scratch inside the
 *    call (copies on `stream`), and the call then synchronises `stream`.  One
 *    exception: page-locked (pinned) host outputs -- csaw_walk's `path`, and
 *    csaw_sample's src / dst / edge_depth on its fused path -- are written by the
 *    kernels directly over the host link, overlapped with the computation.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  csaw_walk
 *    synchronises `stream` once after its seed check and returns after enqueuing
 *    the walk (device buffers); csaw_sample synchronises `stream` once (it must
 *    return *num_edges).
 *  - Ownership: callers own every buffer they pass.  csaw_graph_create copies
 *    the CSR; the graph owns its device copy and its internal scratch (reused
 *    across calls, freed by csaw_graph_destroy).  A graph may be used by one
 *    host thread at a time.
 *  - Errors: every entry point returns a csaw_status, never aborts or prints;
 *    csaw_last_error() returns a thread-local message for the last failure.
 *  - Determinism (R7): every output is a pure function of (graph bytes, bias,
 *    fanout / length, seeds, rng_seed, instance_base + i).  It does not depend
 *    on the stream, GPU count, launch configuration or OOM partitioning.  Draws
 *    are Philox4x32-10 with key (rng_seed lo, rng_seed hi) and counter
 *    (instance, step|depth, slot, purpose<<28 | j<<14 | attempt).
 *  - Vertex ids are uint32; CSAW_NONE (0xFFFFFFFF) marks "no vertex".
 */
#ifndef CSAW_H
#define CSAW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSAW_NONE 0xFFFFFFFFu
#define CSAW_API __attribute__((visibility("default")))

typedef enum {
    CSAW_OK = 0,
    CSAW_ERR_INVALID_ARG = 1,     /* bad parameter (null pointer, k >= 2^14, depth > 255, ...) */
    CSAW_ERR_OUT_OF_RANGE = 2,    /* a seed vertex >= V */
    CSAW_ERR_BAD_GRAPH = 3,       /* CSR validation failed (see csaw_last_error) */
    CSAW_ERR_DEGENERATE_POOL = 4, /* reserved: walks end (pad CSAW_NONE) instead, R20 */
    CSAW_ERR_CAPACITY = 5,        /* output capacity too small; *num_edges = required */
    CSAW_ERR_NO_MEMORY = 6,       /* device / pinned allocation failed or budget exceeded */
    CSAW_ERR_CUDA = 7,            /* CUDA runtime error, or no CUDA device */
    CSAW_ERR_UNSUPPORTED = 8      /* combination not implemented (message says which) */
} csaw_status;

/* Bias selectors: the closed set of VERTEXBIAS / EDGEBIAS / UPDATE triples
 * (Eq. 2-4) the library implements. */
typedef enum {
    CSAW_BIAS_UNIFORM = 0,      /* EdgeBias = 1: unbiased neighbor sampling / simple walk */
    CSAW_BIAS_DEGREE = 1,       /* EdgeBias = deg(u): biased neighbor sampling (Fig. 1) / biased DeepWalk */
    CSAW_BIAS_NODE2VEC = 2,     /* EdgeBias = alpha(prev, u) (R16); walks only.  On a graph with
                                   weights: alpha(prev, u) * w(e) as one fp32 multiply ("depends upon the edge
                                   weight"; R33), float path (R28), step 0 weighted (b = w) */
    CSAW_BIAS_FOREST_FIRE = 3,  /* uniform EdgeBias, per-vertex burn count with P_f (R15); sampling only */
    CSAW_BIAS_LAYER = 4,        /* EdgeBias = deg(u) over the union pool of the frontier (R14); sampling only */
    CSAW_BIAS_MDRW = 5,         /* VertexBias = deg(v), EdgeBias = 1, Update = replace (Fig. 4); walks only */
    /* Table-1 walk variants, uniform proposal u = N(v)[below(U(EDGE), d)]: */
    CSAW_BIAS_MH = 6,           /* Metropolis-Hastings walk: accept iff below(U(ACCEPT), deg u) < deg v, else stay */
    CSAW_BIAS_RESTART = 7,      /* walk with restart: with probability pf return to the start vertex */
    CSAW_BIAS_JUMP = 8,         /* walk with jump: with probability pf jump to below(U(TARGET), V) */
    CSAW_BIAS_SNOWBALL = 9,     /* snowball sampling: every neighbour of every expanded vertex to
                                   `depth` (select-all, R8); fanout ignored (may be NULL); sampling only */
    CSAW_BIAS_WEIGHT = 10       /* EdgeBias = w(e), the graph's fp32 edge weights (Eq. 3, f(e); F real-valued
                                   P:228): walks (biased DeepWalk over weights) and neighbor sampling without
                                   replacement.  Float path (R28): fp32 weights summed in fp64, draw x = r * T with
                                   r = (U >> 11) * 2^-53, region [S_s, S_{s+1}) holding x, zero weights never chosen;
                                   the picks equal the exact fp64 left-to-right definition except for draws within a
                                   few ulps of a region boundary (the summation order differs).  Needs a graph
                                   created with csaw_csr.weights (else INVALID_ARG); in-memory graphs only. */
} csaw_bias_kind;

typedef struct {
    int32_t kind;       /* csaw_bias_kind */
    double p, q;        /* node2vec return / in-out parameters, > 0 */
    double pf;          /* forest-fire burning probability, or restart / jump probability; in [0, 1) */
    int32_t pool_size;  /* MDRW FrontierSize m (2,000), >= 1 */
    int32_t a_max;      /* BRS attempt cap before exact updated sampling (R2); 0 = default 64; even, 2..16382 */
    int32_t migration;  /* collision migration without replacement (§4.2): 0 = bipartite region search
                           (the method), 1 = repeated sampling (Fig. 6(a)), 2 = updated sampling
                           (Fig. 6(b)); 1 and 2 are the paper's baselines, for the Fig. 10-11 ablation */
} csaw_bias;

/* A CSR graph: row_ptr int64[V+1] (row_ptr[0] = 0, non-decreasing, row_ptr[V] = E),
 * col_idx uint32[E] with values < V.  Rows should be sorted ascending without
 * duplicates (node2vec's N(prev) membership test relies on sorted rows; the
 * library checks and reports csaw_graph_info.rows_sorted).  Host or device
 * pointers; copied, never retained.
 * weights: nullable fp32[E], finite and >= 0 (else BAD_GRAPH), aligned with col_idx: the
 * EdgeBias w(e) of CSAW_BIAS_WEIGHT (Eq. 3).  Copied to the device (+ 512 B of
 * zero padding); not supported together with an out-of-memory budget (UNSUPPORTED). */
typedef struct {
    int64_t num_vertices;
    int64_t num_edges;
    const int64_t *row_ptr;
    const uint32_t *col_idx;
    const float *weights;
} csaw_csr;

typedef struct {
    int32_t device;                 /* CUDA device ordinal */
    int64_t device_budget_bytes;    /* 0 = in-memory; > 0 = out-of-memory mode (§5) under this budget */
    int32_t num_partitions;         /* OOM: equal contiguous vertex ranges; 0 = default 4 */
    int32_t max_resident;           /* OOM: partitions resident at once; 0 = default 2 */
    int32_t num_streams;            /* OOM: streams (one kernel per active partition); 0 = default 2 */
    uint32_t flags;                 /* CSAW_GRAPH_* bits */
    int32_t store_device;           /* OOM with CSAW_GRAPH_OOM_PEER_STORE: the GPU whose HBM holds the partition
                                       store (peer access over NVLink is enabled); == device: a same-device
                                       stand-in (tests on one GPU).  Ignored otherwise. */
} csaw_graph_opts;

/* csaw_graph_opts.flags: build the static-bias CTPS cache at creation (in-memory
 * graphs).  cps[e] = sum of deg(col[e']) over e' in [row_ptr[v], e], u64 per CSR
 * entry, plus the per-row count of positive-bias neighbours.  This is the
 * paper's "caching transition probability" (in \begin{comment}; reading
 * R25): degree-biased selections then search the cached prefix (O(log d) reads)
 * instead of re-scanning the neighbour list.  Results are bit-identical (same
 * integer S, same draws). */
#define CSAW_GRAPH_CTPS_CACHE 0x1u
/* csaw_graph_opts.flags, out-of-memory mode only: instead of staging partitions
 * (§5.2 workload-aware scheduling, the default), kernels read col_idx in place
 * from pinned, mapped host memory (zero-copy).  Useful
 * when a step needs one neighbour entry (MDRW, uniform walks); the device then
 * holds only row_ptr + deg + run state.  Every selector is supported.  Without
 * this flag (partition scheduling) csaw_walk implements MDRW, degree and uniform
 * walks and csaw_sample neighbor / forest fire / snowball; others return
 * UNSUPPORTED. */
#define CSAW_GRAPH_OOM_ZEROCOPY 0x2u
/* csaw_graph_opts.flags: csaw_sample always uses the level-synchronous batched
 * driver (one frontier queue mixing all instances) instead of the
 * fused one-warp-per-instance path chosen for small per-instance frontiers.
 * Outputs are identical either way (R7); this flag exists for tests/ablation. */
#define CSAW_GRAPH_SAMPLE_BATCHED 0x4u
/* csaw_graph_opts.flags, OOM ablation (Fig. 13-15; results unchanged):
 * NO_WS  -- partitions are taken in round-robin id order (skipping empty queues)
 *           and evicted first-in-first-out, instead of workload-aware scheduling
 *           (busiest first, residents with work kept);
 * NO_BAL -- every partition kernel of a wave gets the same CTA count instead of
 *           CTAs proportional to its active count. */
#define CSAW_GRAPH_OOM_NO_WS 0x8u
#define CSAW_GRAPH_OOM_NO_BAL 0x10u
/* csaw_graph_opts.flags, with CSAW_GRAPH_CTPS_CACHE: do not build the narrow walk
 * index (paper_2009_09103_b200/csrc/wix.cuh; built by default with the cache when
 * every row total is < 2^32: S as u32 in 128-entry leaves with a col copy, fanout-128
 * internal nodes, a 16 B record and a 512 B head per vertex -- the head holds the
 * record and the row's top index level, or the whole row when d <= 60, at v x 512 B).
 * Degree walks then search the u64 fanout-32 index instead.  Results are identical
 * either way; this flag exists for tests, A/B measurements and memory savings
 * (the index costs 8 (E + 3V) + 528 V bytes). */
#define CSAW_GRAPH_NO_WALK_INDEX 0x20u
/* csaw_graph_opts.flags (in-memory graphs with sorted rows): build per-edge triangle
 * counts tri[e] = |N(v) ∩ N(u)| for every CSR entry e = (v -> u) (one u32 per entry;
 * ignored unless the graph is symmetric).  Integer node2vec walks (R16) then
 * get the row total of each step's CTPS in closed form and scan N(v) only from the end
 * nearer the draw up to its region, instead of merging all of N(v) with N(prev).  The
 * picks are identical (same integer S, same draw).  Reported in csaw_graph_info_t. */
#define CSAW_GRAPH_N2V_TRI 0x40u
/* csaw_graph_opts.flags (in-memory graphs, max degree < 2^24): build next-vertex
 * metadata nmp[e] = row_ptr[u] << 24 | deg(u) for u = col[e] (8 B per CSR entry), so an
 * MDRW step reads the new pool vertex's row and VertexBias together with the
 * picked entry instead of one dependent row_ptr lookup later (degree walks on the u64
 * index, k_walk_cached, use it too).  Results are identical. */
#define CSAW_GRAPH_NEXT_META 0x80u
/* csaw_graph_opts.flags (in-memory graphs): next-vertex records nrec[e] = {u, deg(u),
 * row_ptr[u] lo, hi} for u = col[e] (16 B per CSR entry, best-effort).  An MDRW step
 * then reads the picked entry's vertex and the new pool vertex's row and
 * VertexBias in one 16 B access instead of col[e] and nmp[e] (two random DRAM accesses).
 * Takes precedence over CSAW_GRAPH_NEXT_META for MDRW.  Results are identical. */
#define CSAW_GRAPH_NEXT_RECORD 0x800000u
/* csaw_graph_opts.flags (in-memory graphs, with CSAW_GRAPH_CTPS_CACHE; best-effort): bucketed
 * degree-walk index.  Row v's CTPS [0, T) is cut into nb = ceil(T / 2^k) buckets of width
 * 2^k, k = floor(log2(T / deg(v))) (deg(v) <= nb < 2 deg(v)); bucket b is one 128 B line of 8
 * 16 B entries {S_i, u | k_u << 27, first bucket of u, T_u}, the regions [S_i, S_i + deg(u))
 * meeting [b 2^k, (b + 1) 2^k) in order (a 9th region turns the last entry into a link to the
 * row's CTPS cache).  A degree-walk step is then x = below(U, T), one line at bucket x >> k,
 * the last entry with S_i <= x: the pick and the next vertex's bucket table arrive together
 * -- one dependent DRAM round trip per step instead of two (vertex head, then leaf).  Picks
 * are identical (same integer S, same draw).  Needs every row total < 2^32 - 2 and
 * V < 2^27 - 1; about 128 B x (1..2) per CSR entry.  On a graph with edge weights the flag
 * also builds the float-path twin for CSAW_BIAS_WEIGHT walks (no CTPS cache needed): each row's
 * fp64 prefix of the fp32 weights summed left to right (R28 -- the oracle's sums, bit for bit),
 * buckets of width 2^k (k = floor(log2(T / d)) in [-24, 7]) holding up to 5 candidate regions
 * {S, T_u, u, bucket of u}; a pick is the last positive-weight region with S <= x = r T, so
 * weighted walks match the oracle exactly instead of within the 1e-6 boundary rule. */
#define CSAW_GRAPH_WALK_BUCKETS 0x1000000u
/* csaw_graph_opts.flags (in-memory graphs; built automatically in out-of-memory mode
 * when it fits the budget): chunk-total cache of the degree bias -- for every row of more
 * than 256 candidates, the chunk prefix sums of its CTPS (<= 256 chunks) and its count of
 * positive-bias candidates, E / 64 + 512 u64 in all.  Degree-biased selections read the
 * chunk table instead of scanning the whole pool and rescan one chunk per draw.  Results
 * are identical. */
#define CSAW_GRAPH_CHUNK_CACHE 0x100u
/* csaw_graph_opts.flags (in-memory graphs with sorted rows, max degree < 2^24; used only
 * if the graph is symmetric): node2vec per-edge intersection index.  For every CSR entry
 * e = (prev -> v): the count C of common neighbours N(v) ∩ N(prev), the position of prev in
 * N(v), and the ascending positions in N(v) of the common neighbours (a 128 B record per
 * entry with up to 48 u16 / 24 u32 of them inline, + 2 / 4 B per common-neighbour pair beyond;
 * ~40 GB of device memory with the cfg3 graph).  Integer node2vec walks
 * (R16) then binary-search those positions for the region of the draw (the CTPS
 * is piecewise linear between them) instead of merging N(v) with N(prev): O(log C) reads
 * per step.  Picks are identical.  Best-effort: if the index does not fit, the graph is
 * created without it (csaw_graph_info_t.node2vec_index = 0). */
#define CSAW_GRAPH_N2V_INDEX 0x200u
/* csaw_graph_opts.flags (in-memory graphs): materialised degree bias ebias[e] = deg(col[e]),
 * one u32 per CSR entry (+ padding).  Degree-biased walks without the CTPS cache then stream
 * each pool's biases as 16 B vectors (vscan.cuh) instead of gathering deg[u] per neighbour
 * (one 32 B sector per 4 B): the per-step bias evaluation + warp scan of the CTPS (§4.1,
 * P:477-480) stays, only the gather becomes a coalesced read.  Results are identical. */
#define CSAW_GRAPH_EDGE_BIAS 0x400u
/* csaw_graph_opts.flags -- variant selectors.  Every one leaves the results unchanged (R7);
 * they pick between equivalent data layouts / kernels for tests and A/B measurements:
 *   WALK_NO_HEADS       the walk index without its 512 B vertex heads (walks search records)
 *   WALK_LEAF_64 / _32  walk-index leaf fanout 64 / 32 instead of 128
 *   WALK_GROUP_16 / _8  degree walks on the index with 16 / 8 lanes per walker (leaf >= 64
 *                       for 16) instead of one warp per walker
 *   SAMPLE_NO_HEADS     cached degree / layer sampling pools search the u64 B-tree, not the heads
 *   OOM_NO_CHUNK_CACHE  out-of-memory mode without the automatic chunk-total cache
 *   OOM_ZC_NO_PREFIX    zero-copy OOM mode keeps no col_idx prefix resident (all host reads)
 *   MDRW_GENERIC        MDRW uses the general kernel (shared-memory block totals) for every pool
 *   MDRW_ALT_RECORDS    MDRW pools <= 2,048 slots: 8 B packed slot records row << 24 | degree
 *                       + a vertex-id array instead of 16 B {v, degree, row} records */
/* csaw_graph_opts.flags, out-of-memory mode: the partition store
 * -- the full col_idx the §5 scheduler copies partitions from -- lives in the
 * HBM of opts.store_device instead of pinned host memory.  Partition loads become
 * device-to-device copies over NVLink (cudaMemcpyAsync, ~900 GB/s per direction on
 * NVSwitch vs a PCIe / C2C host link), and with CSAW_GRAPH_OOM_ZEROCOPY the kernels read
 * the peer's memory in place.  The planner, budget and results are unchanged (only the
 * local arena counts against device_budget_bytes).  In-memory graphs ignore it. */
#define CSAW_GRAPH_OOM_PEER_STORE 0x200000u
#define CSAW_GRAPH_WALK_NO_HEADS 0x800u
#define CSAW_GRAPH_WALK_LEAF_64 0x1000u
#define CSAW_GRAPH_WALK_LEAF_32 0x2000u
#define CSAW_GRAPH_WALK_GROUP_16 0x4000u
#define CSAW_GRAPH_WALK_GROUP_8 0x8000u
#define CSAW_GRAPH_SAMPLE_NO_HEADS 0x10000u
#define CSAW_GRAPH_OOM_NO_CHUNK_CACHE 0x20000u
#define CSAW_GRAPH_OOM_ZC_NO_PREFIX 0x40000u
#define CSAW_GRAPH_MDRW_GENERIC 0x80000u
#define CSAW_GRAPH_MDRW_ALT_RECORDS 0x100000u

typedef struct {
    int64_t num_vertices, num_edges;
    int64_t max_degree;
    int64_t nonisolated;            /* vertices with degree > 0 */
    int32_t rows_sorted;            /* 1 if every row is strictly ascending */
    int32_t oom_mode;               /* 1 if created with a device budget */
    int64_t device_bytes;           /* device memory held by the graph (CSR + degree + scratch) */
    int32_t ctps_cache;             /* 1 if the static-bias CTPS cache was built */
    int32_t walk_index_leaf;        /* narrow walk index leaf fanout (32/64/128; 129 = col read after the leaf), 0 = not built */
    double cache_build_ms;          /* device time of the cache build */
    int32_t walk_index_group;       /* lanes per walker of the degree-walk kernel (8 / 16; 32 = one warp per walker) */
    int32_t node2vec_tri;           /* 1 if per-edge triangle counts were built (CSAW_GRAPH_N2V_TRI on a symmetric graph) */
    int32_t walk_index_heads;       /* 1 if the walk index has 512 B vertex heads (degree walks: k_walk_head) */
    int32_t node2vec_index;         /* 1 if the node2vec intersection index was built (CSAW_GRAPH_N2V_INDEX) */
    int32_t has_weights;            /* 1 if the graph carries edge weights (csaw_csr.weights) */
    int32_t edge_bias;              /* 1 if the materialised degree bias was built (CSAW_GRAPH_EDGE_BIAS) */
    int32_t walk_buckets;           /* bucketed walk indices built (CSAW_GRAPH_WALK_BUCKETS): 1 degree, 2 edge weights */
    int32_t reserved0;
} csaw_graph_info_t;

typedef struct csaw_graph csaw_graph;  /* opaque */

/* Counters of the last csaw_sample / csaw_walk on a graph (SURVEY §5 "metrics"). */
typedef struct {
    uint64_t sampled_edges;         /* SEPS numerator (R30) */
    uint64_t pools;                 /* selection pools processed (frontier entries / walk steps) */
    uint64_t neighbours_scanned;    /* candidates whose bias was evaluated (pass 1 of the CTPS build) */
    uint64_t partition_loads;       /* OOM: partition transfers (Fig. 15) */
    uint64_t h2d_bytes;             /* OOM: bytes copied from the partition store (host, or the peer GPU) */
    uint64_t cache_probes;          /* CTPS-cache entries read by the searches (CSAW_GRAPH_CTPS_CACHE) */
    uint64_t draws;                 /* random draws consumed by without-replacement selections (Fig. 11) */
    uint64_t kernel_launches;       /* kernels this library launched for the call */
    uint64_t hot_launches;          /* launches of the selection ("hot") kernel */
    double kernel_ms;               /* device time, first launch -> last completion (CUDA events) */
    double hot_kernel_ms;           /* summed device time of the hot-kernel launches (CUDA events) */
    double transfer_ms;             /* OOM: partition-transfer time */
    uint64_t index_bytes;           /* bytes of walk-index records, nodes, leaves and col entries read (narrow walk index) */
} csaw_run_stats;

/* Create a graph on opt->device (opt may be NULL: device 0, in-memory).
 * Validates the CSR (row_ptr monotone, row_ptr[V] = E, col < V) on the device,
 * builds deg[v] = row_ptr[v+1]-row_ptr[v] (u32).  Errors: INVALID_ARG (null /
 * negative sizes / V >= 2^32-1), BAD_GRAPH (incl. a negative or non-finite weight),
 * UNSUPPORTED (weights with a device budget), NO_MEMORY, CUDA. */
CSAW_API csaw_status csaw_graph_create(const csaw_csr *csr, const csaw_graph_opts *opt, csaw_graph **out);
CSAW_API csaw_status csaw_graph_destroy(csaw_graph *g);
CSAW_API csaw_status csaw_graph_info(const csaw_graph *g, csaw_graph_info_t *out);

/* Upper bound on the number of sampled edges csaw_sample can emit for
 * neighbor / layer sampling: n * sum_d prod_{d'<=d} fanout[d'] (neighbor) or
 * n * sum_d fanout[d] (layer).  Forest fire has no fixed bound: returns an
 * estimate from the burn law, and csaw_sample reports CSAW_ERR_CAPACITY with
 * the exact requirement if it is too small. */
CSAW_API csaw_status csaw_sample_capacity(const csaw_bias *bias, const int32_t *fanout, int32_t depth,
                                          int64_t n_instances, int64_t *capacity);

/*
 * Traversal sampling (neighbor / forest fire / layer), Fig. 2(b) main loop
 * with Select = ITS over an integer CTPS (Eq. 1) and
 * without-replacement collision migration by bipartite region search (§4.2,
 * P:514-565) with bitmap collision detection.  UPDATE appends every
 * not-yet-visited pick to the instance's next frontier (R9).
 *
 *   bias          kind UNIFORM, DEGREE, FOREST_FIRE or LAYER (host pointer)
 *   fanout        host int32[depth]: NeighborSize per depth (ignored for FOREST_FIRE), 0 <= fanout < 2^14
 *   depth         1..255
 *   seeds         uint32[n_instances]: one seed vertex per instance (host or device)
 *   instance_base global id of seeds[0] (multi-GPU sharding, R7)
 *   offsets       uint64[n_instances+1]: instance i's edges are [offsets[i], offsets[i+1])
 *   src,dst       uint32[capacity]; edge_depth uint8[capacity] (1..depth)
 *                 per instance in canonical order (depth, src, dst) (R11)
 *   num_edges     host int64*: total edges written (or required, on CAPACITY)
 * Returns OUT_OF_RANGE if a seed >= V (nothing written), CAPACITY if the
 * output does not fit (offsets written, edges not written).
 */
CSAW_API csaw_status csaw_sample(const csaw_graph *g, const csaw_bias *bias, const int32_t *fanout, int32_t depth,
                                 const uint32_t *seeds, int64_t n_instances, uint64_t instance_base,
                                 uint64_t rng_seed, uint64_t *offsets, uint32_t *src, uint32_t *dst,
                                 uint8_t *edge_depth, int64_t capacity, int64_t *num_edges, void *stream);

/*
 * Random walks, with replacement: DEGREE (biased DeepWalk),
 * UNIFORM (DeepWalk), NODE2VEC (step 0 uniform, R16), MDRW
 * (multi-dimensional random walk, Fig. 4).
 *   DEGREE / UNIFORM / NODE2VEC: seeds uint32[n_walkers]; path uint32[n_walkers][length+1],
 *     path[w][0] = seeds[w]; a walker at a vertex with no positive-bias
 *     neighbour stops and the rest of its row is CSAW_NONE (R20).
 *   MDRW: seeds uint32[n_walkers][pool_size] (the instance's initial pool, slot
 *     order); path uint32[n_walkers][length][2] = the (v, u) edge sampled at each step.
 *   WEIGHT: as DEGREE with EdgeBias = w(e) (graphs created with weights); MH / RESTART /
 *     JUMP: the path is the sequence of positions -- a rejected Metropolis-Hastings proposal
 *     repeats the current vertex, a restart / jump is the next entry like an edge step (the
 *     path is not an edge list for these three).
 * Returns OUT_OF_RANGE if a seed >= V (checked on the device before any walk kernel;
 * the call then synchronises `stream` once, nothing is written to path).
 * csaw_run_stats.sampled_edges counts length per walker (R30) even for a walk that ended
 * early (R20, padded with CSAW_NONE); for degree / uniform / node2vec / weight walks .pools
 * counts the transitions actually taken.
 */
CSAW_API csaw_status csaw_walk(const csaw_graph *g, const csaw_bias *bias, int32_t length,
                               const uint32_t *seeds, int64_t n_walkers, uint64_t instance_base,
                               uint64_t rng_seed, uint32_t *path, void *stream);

/* Counters of the last run on g.  Synchronises on the call's completion event. */
CSAW_API csaw_status csaw_stats(const csaw_graph *g, csaw_run_stats *out);

/* Thread-local description of the last error ("" if none). */
CSAW_API const char *csaw_last_error(void);

/* Library version string, e.g. "csaw-b200 0.1 sm_100a". */
CSAW_API const char *csaw_version(void);

/* Test hook: Philox4x32-10 on the device for n counters (ctr uint32[n][4],
 * key uint32[2], out uint32[n][4]; host or device pointers).  Lets tests pin
 * the device generator against the Random123 KATs and cuRAND's device Philox. */
CSAW_API csaw_status csaw_philox(const uint32_t *ctr, const uint32_t *key, uint32_t *out, int64_t n);

/* Test hook: compares the library's device Philox with cuRAND's
 * curand_Philox4x32_10 on n pseudo-random counters; *mismatches = count. */
CSAW_API csaw_status csaw_selftest_curand(int64_t n, int64_t *mismatches);

#ifdef __cplusplus
}
#endif
#endif /* CSAW_H */
