/*
 * C-SAW CPU ORACLE — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, single-threaded C implementation of what C-SAW's hot path
 * computes (arXiv 2009.09103, "C-SAW: A Framework for Graph Sampling and Random
 * Walk on GPUs").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant generator with the CUDA library under
 * paper_2009_09103_b200/csrc/, and neither includes the other.
 *
 * Citations: "P:n" = line n of the paper's LaTeX; "R<n>" = reading
 * n of DESIGN.md §3 (where the paper is silent, garbled or self-inconsistent).
 *
 * Conventions (all exact integer arithmetic for integer biases, R1):
 *   - CTPS in integers: S[0] = 0, S[i+1] = S[i] + b[i], T = S[n]   (Eq. 1; R5)
 *     F = S/T is never formed; a draw is x in [0, T)              (R6)
 *   - its(S, x) = the unique s with S[s] <= x < S[s+1]              (R4)
 *   - draws: Philox4x32-10 (Salmon et al., SC'11) keyed by the run's rng_seed,
 *     counter (instance, step|depth, slot, purpose<<28 | j<<14 | attempt) (R7)
 *   - below(U, M) = floor(U * M / 2^64)                             (R7)
 *
 * Pins: tests/test_oracle_*.py (KATs, paper worked examples, closed forms,
 * brute-force enumeration, invariants).  Functions with no pin are marked
 * "parity unpinned" here and in DESIGN.md.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORACLE_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Random123 round function; R7).  Pinned by the Random123    */
/* known-answer vectors in tests/golden/philox_kat.txt.                      */
/* ------------------------------------------------------------------------- */
ORACLE_EXPORT void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Purposes of a draw (R7). */
enum { P_EDGE = 0, P_VERTEX = 1, P_BURN = 2, P_ACCEPT = 3, P_JUMP = 4, P_TARGET = 5 };

/* U(i, t, slot, word3) = o0 | o1 << 32 of philox((i, t, slot, word3); key(seed)). */
static uint64_t draw_u64(uint64_t seed, uint32_t i, uint32_t t, uint32_t slot, uint32_t word3, uint32_t *o0_out)
{
    uint32_t ctr[4] = { i, t, slot, word3 };
    uint32_t key[2] = { (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32) };
    uint32_t o[4];
    oracle_philox4x32_10(ctr, key, o);
    if (o0_out) *o0_out = o[0];
    return (uint64_t)o[0] | ((uint64_t)o[1] << 32);
}

static uint32_t word3_of(uint32_t purpose, uint32_t j, uint32_t a)
{
    return (purpose << 28) | (j << 14) | a;
}

/* below(U, M) = floor(U * M / 2^64): a uniform integer in [0, M) (R7). */
ORACLE_EXPORT uint64_t oracle_below(uint64_t U, uint64_t M)
{
    unsigned __int128 p = (unsigned __int128)U * (unsigned __int128)M;
    return (uint64_t)(p >> 64);
}

/* ------------------------------------------------------------------------- */
/* CTPS and inverse transform sampling (Eq. 1).                   */
/* ------------------------------------------------------------------------- */

/* S[0..n] from b[0..n): S[0] = 0, S[i+1] = S[i] + b[i] (R5). */
ORACLE_EXPORT void oracle_prefix(const uint32_t *b, int64_t n, uint64_t *S)
{
    S[0] = 0;
    for (int64_t i = 0; i < n; i++) S[i + 1] = S[i] + (uint64_t)b[i];
}

/* its(S, x): the unique s with S[s] <= x < S[s+1], 0 <= x < S[n].
 * A linear scan: the plain definition, no search structure. */
ORACLE_EXPORT int64_t oracle_its(const uint64_t *S, int64_t n, uint64_t x)
{
    for (int64_t s = 0; s < n; s++)
        if (S[s] <= x && x < S[s + 1]) return s;
    return -1;  /* x >= T: outside the CTPS */
}

/* ------------------------------------------------------------------------- */
/* Selection without replacement with bipartite region search                */
/* (§4.2 boxed steps 1-5; Theorem 2).                  */
/* ------------------------------------------------------------------------- */
typedef struct {
    uint64_t seed;     /* rng_seed */
    uint32_t inst;     /* global instance id */
    uint32_t t;        /* depth (sampling) */
    uint32_t slot;     /* frontier vertex id, or 0xFFFFFFFF for a layer pool */
} draw_ctx;

static int in_list(const int64_t *list, int64_t cnt, int64_t v)
{
    for (int64_t i = 0; i < cnt; i++) if (list[i] == v) return 1;
    return 0;
}

static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* Steps (3)-(5) of the box for one pre-selected candidate s with
 * region [l, h) = [S[s], S[s+1]) and delta = b[s]: x2 is a draw over the CTPS
 * with that region removed, [0, T - delta).  Left part (0, l): y = x2; right
 * part (h, 1): y = x2 + delta ("update r to r + delta").  Returns its(S, y).
 * Theorem 2 says this equals ITS over the updated CTPS (Fig. 6(b))
 * at the same survivor position x2 -- pinned exhaustively in
 * tests/test_oracle_select.py. */
ORACLE_EXPORT int64_t oracle_brs_step(const uint64_t *S, const uint32_t *b, int64_t n, int64_t s, uint64_t x2)
{
    uint64_t L = S[s], d = (uint64_t)b[s];
    uint64_t y = (x2 < L) ? x2 : x2 + d;
    return oracle_its(S, n, y);
}

/*
 * select_wor: k distinct picks from b[0..n), in pick order j = 0..k-1.
 * Returns the number of picks.  Sequential semantics: pick j sees picks < j
 * (R3).  Steps:
 *   (1)(2) s = its(S, below(U(j,a), T)); accept if not taken
 *   (3)    fresh x' = below(U(j,a+1), T - b[s]) over the space with the
 *          taken region [S[s], S[s+1]) removed (R1 fresh draw, Theorem 2)
 *   (4)(5) y = x' if x' < S[s] (left part (0,l)) else x' + b[s] (right part
 *          (h,1), "r + delta"); s = its(S, y); accept if not taken, else
 *          back to (1)
 *   after a_max attempts: exact updated sampling (Fig. 6(b)) over
 *   the untaken positive-bias candidates with draw U(j, a_max) (R2).
 * If k >= #positive-bias candidates: all of them, ascending (R8).
 * attempts_out (nullable) accumulates the number of draws used.
 */
/* Collision migration mode (§4.2): 0 = bipartite region search (the method),
 * 1 = repeated sampling (Fig. 6(a)), 2 = updated sampling (Fig. 6(b),
 * P:508-511).  The baselines exist for the Fig. 10-11 ablation. Single-threaded
 * oracle: a process-wide setting. */
static int g_migration = 0;
ORACLE_EXPORT void oracle_set_migration(int32_t mode) { g_migration = mode; }

/* Exact updated sampling (Fig. 6(b)): rebuild the CTPS over the positive-bias,
 * untaken candidates (ascending) and search it with U. */
static int64_t updated_pick(const uint32_t *b, int64_t n, const int64_t *picks, int64_t taken, uint64_t U)
{
    int64_t nsv = 0;
    int64_t *sv = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    uint32_t *b2 = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; i++)
        if (b[i] > 0 && !in_list(picks, taken, i)) { sv[nsv] = i; b2[nsv] = b[i]; nsv++; }
    uint64_t *S2 = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(nsv + 1));
    oracle_prefix(b2, nsv, S2);
    int64_t s = sv[oracle_its(S2, nsv, oracle_below(U, S2[nsv]))];
    free(S2); free(b2); free(sv);
    return s;
}

/*
 * select_wor: k distinct picks from b[0..n), in pick order j = 0..k-1.
 * Returns the number of picks.  Sequential semantics: pick j sees picks < j
 * (R3).  Steps (mode 0, bipartite region search):
 *   (1)(2) s = its(S, below(U(j,a), T)); accept if not taken
 *   (3)    fresh x' = below(U(j,a+1), T - b[s]) over the space with the
 *          taken region [S[s], S[s+1]) removed (R1 fresh draw, Theorem 2)
 *   (4)(5) y = x' if x' < S[s] (left part (0,l)) else x' + b[s] (right part
 *          (h,1), "r + delta"); s = its(S, y); accept if not taken, else
 *          back to (1)
 *   after a_max attempts: exact updated sampling (Fig. 6(b)) over
 *   the untaken positive-bias candidates with draw U(j, a_max) (R2).
 * Mode 1 (repeated sampling): redraw (1)(2) until untaken, same cap.
 * Mode 2 (updated sampling): every pick is updated sampling with U(j, 0).
 * If k >= #positive-bias candidates: all of them, ascending (R8).
 * attempts_out (nullable) accumulates the number of draws used.
 */
ORACLE_EXPORT int64_t oracle_select_wor(const uint32_t *b, int64_t n, int64_t k,
                                        uint64_t seed, uint32_t inst, uint32_t t, uint32_t slot,
                                        int32_t a_max, int64_t *picks, int64_t *attempts_out)
{
    int64_t npos = 0;
    for (int64_t i = 0; i < n; i++) if (b[i] > 0) npos++;
    if (k <= 0 || npos == 0) return 0;
    if (k >= npos) {
        int64_t c = 0;
        for (int64_t i = 0; i < n; i++) if (b[i] > 0) picks[c++] = i;
        return c;
    }
    uint64_t *S = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(n + 1));
    oracle_prefix(b, n, S);
    uint64_t T = S[n];
    int64_t taken = 0;
    for (int64_t j = 0; j < k; j++) {
        uint32_t a = 0;
        int64_t s;
        if (g_migration == 2) {
            s = updated_pick(b, n, picks, taken, draw_u64(seed, inst, t, slot, word3_of(P_EDGE, (uint32_t)j, 0), 0));
            a = 1;
        } else {
            for (;;) {
                s = oracle_its(S, n, oracle_below(draw_u64(seed, inst, t, slot, word3_of(P_EDGE, (uint32_t)j, a), 0), T));
                a += 1;
                if (!in_list(picks, taken, s)) break;
                if (g_migration == 0) {
                    uint64_t x2 = oracle_below(draw_u64(seed, inst, t, slot, word3_of(P_EDGE, (uint32_t)j, a), 0), T - (uint64_t)b[s]);
                    a += 1;
                    s = oracle_brs_step(S, b, n, s, x2);
                    if (!in_list(picks, taken, s)) break;
                }
                if ((int32_t)a >= a_max) {
                    s = updated_pick(b, n, picks, taken,
                                     draw_u64(seed, inst, t, slot, word3_of(P_EDGE, (uint32_t)j, (uint32_t)a_max), 0));
                    a += 1;
                    break;
                }
            }
        }
        if (attempts_out) *attempts_out += a;
        picks[taken++] = s;
    }
    free(S);
    return taken;
}

/* ------------------------------------------------------------------------- */
/* Graph helpers                                                             */
/* ------------------------------------------------------------------------- */
typedef struct {
    const int64_t *row_ptr;   /* [V+1] */
    const uint32_t *col;      /* [E], rows sorted ascending */
    int64_t V;
} csr_t;

static int64_t deg_of(const csr_t *g, uint32_t v) { return g->row_ptr[v + 1] - g->row_ptr[v]; }

/* sampled-edge record; canonical order (depth, src, dst) (R11) */
typedef struct { uint32_t src, dst; uint8_t depth; } edge_t;

static int cmp_edge(const void *a, const void *b)
{
    const edge_t *x = (const edge_t *)a, *y = (const edge_t *)b;
    if (x->depth != y->depth) return (x->depth > y->depth) - (x->depth < y->depth);
    if (x->src != y->src) return (x->src > y->src) - (x->src < y->src);
    return (x->dst > y->dst) - (x->dst < y->dst);
}

typedef struct { int64_t *v; int64_t n, cap; } vec_t;
static void vpush(vec_t *a, int64_t x)
{
    if (a->n == a->cap) { a->cap = a->cap ? 2 * a->cap : 16; a->v = (int64_t *)realloc(a->v, sizeof(int64_t) * (size_t)a->cap); }
    a->v[a->n++] = x;
}
typedef struct { edge_t *e; int64_t n, cap; } evec_t;
static void epush(evec_t *a, uint32_t s, uint32_t d, uint8_t dep)
{
    if (a->n == a->cap) { a->cap = a->cap ? 2 * a->cap : 16; a->e = (edge_t *)realloc(a->e, sizeof(edge_t) * (size_t)a->cap); }
    a->e[a->n].src = s; a->e[a->n].dst = d; a->e[a->n].depth = dep; a->n++;
}

/* sort + unique in place */
static void vsort_unique(vec_t *a)
{
    if (a->n == 0) return;
    qsort(a->v, (size_t)a->n, sizeof(int64_t), cmp_i64);
    int64_t w = 1;
    for (int64_t i = 1; i < a->n; i++) if (a->v[i] != a->v[w - 1]) a->v[w++] = a->v[i];
    a->n = w;
}

static int64_t emit_edges(evec_t *out, uint32_t *src, uint32_t *dst, uint8_t *dep, int64_t cap)
{
    if (out->n > 0) qsort(out->e, (size_t)out->n, sizeof(edge_t), cmp_edge);
    if (out->n > cap) return -out->n;
    for (int64_t i = 0; i < out->n; i++) { src[i] = out->e[i].src; dst[i] = out->e[i].dst; dep[i] = out->e[i].depth; }
    return out->n;
}

/* Forest-fire burn threshold theta = floor(pf * 2^32) (R15). */
ORACLE_EXPORT uint64_t oracle_ff_theta(double pf)
{
    return (uint64_t)floor(pf * 4294967296.0);
}

/* Forest-fire burn count for frontier vertex v: consecutive successes of
 * o0 < theta, truncated at deg(v) (R15). */
ORACLE_EXPORT int64_t oracle_ff_burn(uint64_t seed, uint32_t inst, uint32_t depth, uint32_t v,
                                     int64_t deg, double pf)
{
    uint64_t theta = oracle_ff_theta(pf);
    int64_t x = 0;
    while (x < deg) {
        uint32_t o0;
        draw_u64(seed, inst, depth, v, (P_BURN << 28) | (uint32_t)x, &o0);
        if ((uint64_t)o0 < theta) x++; else break;
    }
    return x;
}

/*
 * Traversal sampling for one instance: neighbor sampling (bias 0 = uniform,
 * 1 = degree of the neighbour, R12), forest fire (kind 2, uniform bias, k
 * per vertex from oracle_ff_burn) and snowball (kind 3: every
 * neighbour of every expanded vertex, i.e. k = deg(v) -> select-all, R8).  Fig. 2(b) main loop:
 * FrontierPool <- seeds; per depth: NeighborPool = N(v) in CSR order, EdgeBias,
 * Select (select_wor), Update = post-filter of visited vertices (R9),
 * Sampled <- picks.  Each v in sorted(F) is one pool.
 * Returns #edges (canonical order), or -(#edges) if cap is too small.
 */
ORACLE_EXPORT int64_t oracle_select_wor_float(const float *b, int64_t n, int64_t k, uint64_t seed, uint32_t inst,
                                              uint32_t t, uint32_t slot, int32_t a_max, int64_t *picks,
                                              double *margin);   /* defined with the float path below */

static int64_t neighbor_sample_core(const int64_t *row_ptr, const uint32_t *col, const float *w, int64_t V,
                                    int32_t kind, const int32_t *fanout, int32_t depth, double pf,
                                    uint32_t seed_vertex, uint32_t inst, uint64_t rng_seed, int32_t a_max,
                                    uint32_t *src, uint32_t *dst, uint8_t *edepth, int64_t cap,
                                    int64_t *attempts_out, double *margin_out)
{
    csr_t g = { row_ptr, col, V };
    if (margin_out) *margin_out = 1.0;
    vec_t visited = {0}, F = {0}, nxt = {0};
    evec_t out = {0};
    vpush(&visited, seed_vertex);
    vpush(&F, seed_vertex);
    for (int32_t d = 0; d < depth; d++) {
        nxt.n = 0;
        for (int64_t fi = 0; fi < F.n; fi++) {          /* F is sorted ascending */
            uint32_t v = (uint32_t)F.v[fi];
            int64_t n = deg_of(&g, v);
            const uint32_t *pool = col + row_ptr[v];
            uint32_t *b = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
            for (int64_t i = 0; i < n; i++)
                b[i] = (kind == 1) ? (uint32_t)deg_of(&g, pool[i]) : 1u;
            int64_t k = (kind == 2) ? oracle_ff_burn(rng_seed, inst, (uint32_t)d, v, n, pf)
                      : (kind == 3) ? n : fanout[d];
            int64_t *picks = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
            int64_t np;
            if (w) {   /* EdgeBias = w(e) (Eq. 3): float path (R28) */
                double mg = 1.0;
                np = oracle_select_wor_float(w + row_ptr[v], n, k, rng_seed, inst, (uint32_t)d, v, a_max, picks, &mg);
                if (margin_out && mg < *margin_out) *margin_out = mg;
            } else {
                np = oracle_select_wor(b, n, k, rng_seed, inst, (uint32_t)d, v, a_max, picks, attempts_out);
            }
            for (int64_t p = 0; p < np; p++) {
                uint32_t u = pool[picks[p]];
                epush(&out, v, u, (uint8_t)(d + 1));
                if (!in_list(visited.v, visited.n, u)) vpush(&nxt, u);   /* Update (R9) */
            }
            free(picks); free(b);
        }
        vsort_unique(&nxt);                                   /* set semantics (R10) */
        for (int64_t i = 0; i < nxt.n; i++) vpush(&visited, nxt.v[i]);
        F.n = 0;
        for (int64_t i = 0; i < nxt.n; i++) vpush(&F, nxt.v[i]);
        if (F.n == 0) break;
    }
    int64_t r = emit_edges(&out, src, dst, edepth, cap);
    free(visited.v); free(F.v); free(nxt.v); free(out.e);
    return r;
}

ORACLE_EXPORT int64_t oracle_neighbor_sample(const int64_t *row_ptr, const uint32_t *col, int64_t V,
                                             int32_t kind, const int32_t *fanout, int32_t depth, double pf,
                                             uint32_t seed_vertex, uint32_t inst, uint64_t rng_seed, int32_t a_max,
                                             uint32_t *src, uint32_t *dst, uint8_t *edepth, int64_t cap,
                                             int64_t *attempts_out)
{
    return neighbor_sample_core(row_ptr, col, NULL, V, kind, fanout, depth, pf, seed_vertex, inst, rng_seed, a_max,
                                src, dst, edepth, cap, attempts_out, NULL);
}

/* Edge-weight neighbor sampling (EdgeBias = w(e), Eq. 3): the traversal
 * of oracle_neighbor_sample with fanout[d] picks per pool from
 * oracle_select_wor_float over the row's weights.  *margin_out (nullable) = the
 * minimum boundary margin over every draw of the instance (R28). */
ORACLE_EXPORT int64_t oracle_weight_sample(const int64_t *row_ptr, const uint32_t *col, const float *w, int64_t V,
                                           const int32_t *fanout, int32_t depth, uint32_t seed_vertex, uint32_t inst,
                                           uint64_t rng_seed, int32_t a_max, uint32_t *src, uint32_t *dst,
                                           uint8_t *edepth, int64_t cap, double *margin_out)
{
    return neighbor_sample_core(row_ptr, col, w, V, 0, fanout, depth, 0.0, seed_vertex, inst, rng_seed, a_max,
                                src, dst, edepth, cap, NULL, margin_out);
}

/*
 * Layer sampling for one instance (Table 1 "per layer"; R14):
 * per depth the pool is the multiset union of N(v) over v in sorted(F), in that
 * order; bias = deg(u); fanout[d] distinct pool entries per layer; draws keyed
 * with slot 0xFFFFFFFF.  Update as neighbor sampling.
 */
ORACLE_EXPORT int64_t oracle_layer_sample(const int64_t *row_ptr, const uint32_t *col, int64_t V,
                                          const int32_t *fanout, int32_t depth,
                                          uint32_t seed_vertex, uint32_t inst, uint64_t rng_seed, int32_t a_max,
                                          uint32_t *src, uint32_t *dst, uint8_t *edepth, int64_t cap,
                                          int64_t *attempts_out)
{
    csr_t g = { row_ptr, col, V };
    vec_t visited = {0}, F = {0}, nxt = {0};
    evec_t out = {0};
    vpush(&visited, seed_vertex);
    vpush(&F, seed_vertex);
    for (int32_t d = 0; d < depth; d++) {
        nxt.n = 0;
        int64_t n = 0;
        for (int64_t fi = 0; fi < F.n; fi++) n += deg_of(&g, (uint32_t)F.v[fi]);
        uint32_t *pv = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
        uint32_t *pu = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
        uint32_t *b = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
        int64_t c = 0;
        for (int64_t fi = 0; fi < F.n; fi++) {
            uint32_t v = (uint32_t)F.v[fi];
            for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++) {
                pv[c] = v; pu[c] = col[e]; b[c] = (uint32_t)deg_of(&g, col[e]); c++;
            }
        }
        int64_t *picks = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
        int64_t np = oracle_select_wor(b, n, fanout[d], rng_seed, inst, (uint32_t)d, 0xFFFFFFFFu, a_max, picks, attempts_out);
        for (int64_t p = 0; p < np; p++) {
            uint32_t v = pv[picks[p]], u = pu[picks[p]];
            epush(&out, v, u, (uint8_t)(d + 1));
            if (!in_list(visited.v, visited.n, u)) vpush(&nxt, u);
        }
        free(picks); free(b); free(pu); free(pv);
        vsort_unique(&nxt);
        for (int64_t i = 0; i < nxt.n; i++) vpush(&visited, nxt.v[i]);
        F.n = 0;
        for (int64_t i = 0; i < nxt.n; i++) vpush(&F, nxt.v[i]);
        if (F.n == 0) break;
    }
    int64_t r = emit_edges(&out, src, dst, edepth, cap);
    free(visited.v); free(F.v); free(nxt.v); free(out.e);
    return r;
}

/* ------------------------------------------------------------------------- */
/* Random walks (with replacement; Theorem 1 transition)   */
/* ------------------------------------------------------------------------- */

/* One step of a degree / uniform walk at vertex v (bias 1 = degree of the
 * neighbour, 0 = uniform).  Returns the next vertex or
 * 0xFFFFFFFF if the pool has total bias 0 (R20). */
ORACLE_EXPORT uint32_t oracle_walk_step(const int64_t *row_ptr, const uint32_t *col, int64_t V,
                                        int32_t kind, uint32_t v, uint32_t inst, uint32_t t, uint64_t rng_seed)
{
    csr_t g = { row_ptr, col, V };
    int64_t n = deg_of(&g, v);
    const uint32_t *pool = col + row_ptr[v];
    uint64_t *S = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(n + 1));
    S[0] = 0;
    for (int64_t i = 0; i < n; i++) S[i + 1] = S[i] + (kind == 1 ? (uint64_t)deg_of(&g, pool[i]) : 1u);
    uint64_t T = S[n];
    uint32_t next = 0xFFFFFFFFu;
    if (T > 0) {
        uint64_t x = oracle_below(draw_u64(rng_seed, inst, t, 0, word3_of(P_EDGE, 0, 0), 0), T);
        next = pool[oracle_its(S, n, x)];
    }
    free(S);
    return next;
}

/* Degree-biased walk (biased DeepWalk) or simple walk:
 * path[0] = s0, path[t+1] = step(path[t]); padded with 0xFFFFFFFF after a dead end. */
ORACLE_EXPORT void oracle_walk(const int64_t *row_ptr, const uint32_t *col, int64_t V,
                               int32_t kind, int32_t length, uint32_t s0, uint32_t inst, uint64_t rng_seed,
                               uint32_t *path)
{
    path[0] = s0;
    for (int32_t t = 0; t < length; t++) {
        uint32_t v = path[t];
        path[t + 1] = (v == 0xFFFFFFFFu) ? 0xFFFFFFFFu
                                         : oracle_walk_step(row_ptr, col, V, kind, v, inst, (uint32_t)t, rng_seed);
    }
}

/*
 * Table-1 walk variants, one step at v, uniform proposal
 * u = N(v)[below(U(i,t,0,EDGE), d)] (the simple walk's draw):
 *   kind 6 Metropolis-Hastings walk: accept u iff
 *          below(U(i,t,0,ACCEPT), deg u) < deg v  (probability min(1, deg v / deg u)),
 *          else stay at v;
 *   kind 7 random walk with restart: with probability pr (o0 of
 *          U(i,t,0,JUMP) < floor(pr 2^32)) return to the walk's start s0;
 *   kind 8 random walk with jump: with the same test, jump to the
 *          vertex below(U(i,t,0,TARGET), V).
 * A vertex without neighbours ends the walk (R20) unless a restart / jump fires.
 */
ORACLE_EXPORT uint32_t oracle_walk_variant_step(const int64_t *row_ptr, const uint32_t *col, int64_t V,
                                                int32_t kind, double pr, uint32_t s0, uint32_t v,
                                                uint32_t inst, uint32_t t, uint64_t rng_seed)
{
    csr_t g = { row_ptr, col, V };
    if (kind == 7 || kind == 8) {
        uint32_t o0;
        draw_u64(rng_seed, inst, t, 0, word3_of(P_JUMP, 0, 0), &o0);
        if ((uint64_t)o0 < (uint64_t)floor(pr * 4294967296.0)) {
            if (kind == 7) return s0;
            return (uint32_t)oracle_below(draw_u64(rng_seed, inst, t, 0, word3_of(P_TARGET, 0, 0), 0), (uint64_t)V);
        }
    }
    int64_t d = deg_of(&g, v);
    if (d == 0) return 0xFFFFFFFFu;
    uint32_t u = col[row_ptr[v] + (int64_t)oracle_below(draw_u64(rng_seed, inst, t, 0, word3_of(P_EDGE, 0, 0), 0), (uint64_t)d)];
    if (kind == 6) {
        uint64_t du = (uint64_t)deg_of(&g, u);
        uint64_t a = oracle_below(draw_u64(rng_seed, inst, t, 0, word3_of(P_ACCEPT, 0, 0), 0), du);
        if (!(a < (uint64_t)d)) return v;   /* rejected: stay */
    }
    return u;
}

ORACLE_EXPORT void oracle_walk_variant(const int64_t *row_ptr, const uint32_t *col, int64_t V, int32_t kind,
                                       double pr, int32_t length, uint32_t s0, uint32_t inst, uint64_t rng_seed,
                                       uint32_t *path)
{
    path[0] = s0;
    for (int32_t t = 0; t < length; t++) {
        uint32_t v = path[t];
        path[t + 1] = (v == 0xFFFFFFFFu) ? 0xFFFFFFFFu
            : oracle_walk_variant_step(row_ptr, col, V, kind, pr, s0, v, inst, (uint32_t)t, rng_seed);
    }
}

/*
 * Float-bias inverse transform sampling (R28; Eq. 1 P:224-247 with real-valued
 * biases, "F is the prefix sum normalised"): b[0..n) fp32 (non-negative,
 * finite), S[0] = 0, S[i+1] = S[i] + (double)b[i] summed left to right in fp64,
 * T = S[n]; r = (U >> 11) * 2^-53 in [0, 1); x = r * T (one fp64 multiply);
 * s = max{i < n : S[i] <= x, b[i] > 0} (the region [S[s], S[s+1]) holding x;
 * zero-width regions are never chosen, R4).  *margin (nullable) receives
 * min_{0<i<n} |x - S[i]| / T: how close the draw came to an interior boundary,
 * relative to T (the checker's 1e-6 rule).  Returns -1 if T == 0.
 * Pinned by hand-computed draws at, and one ulp either side of, a boundary
 * (tests/test_oracle_float.py).
 */
ORACLE_EXPORT int64_t oracle_select_float(const float *b, int64_t n, uint64_t U, double *margin)
{
    if (margin) *margin = 1.0;
    double *S = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    S[0] = 0.0;
    for (int64_t i = 0; i < n; i++) S[i + 1] = S[i] + (double)b[i];
    double T = S[n];
    int64_t s = -1;
    if (T > 0.0) {
        double r = (double)(U >> 11) * (1.0 / 9007199254740992.0);
        double x = r * T;
        for (int64_t i = 0; i < n; i++) if (S[i] <= x && b[i] > 0.0f) s = i;
        if (margin) {
            double mg = 1.0;
            for (int64_t i = 1; i < n; i++) { double dd = fabs(x - S[i]) / T; if (dd < mg) mg = dd; }
            *margin = mg;
        }
    }
    free(S);
    return s;
}

/* ------------------------------------------------------------------------- */
/* Edge-weight bias (EdgeBias = f(e), Eq. 3; "F is real-valued",   */
/* P:228): the float path of reading R28 for walks and without-replacement  */
/* sampling.                                                                 */
/* ------------------------------------------------------------------------- */

/* r = (U >> 11) * 2^-53 in [0, 1) (R28). */
static double unit_r(uint64_t U) { return (double)(U >> 11) * (1.0 / 9007199254740992.0); }

/* its over an fp64 prefix: max{i < n : S[i] <= x, b[i] > 0}, -1 if none (R4, R28). */
static int64_t its_float(const double *S, const float *b, int64_t n, double x)
{
    int64_t s = -1;
    for (int64_t i = 0; i < n; i++) if (S[i] <= x && b[i] > 0.0f) s = i;
    return s;
}

/* min_{0<i<n} |x - S[i]| / T, the checker's boundary margin (R28). */
static double margin_float(const double *S, int64_t n, double x, double T)
{
    double mg = 1.0;
    for (int64_t i = 1; i < n; i++) { double dd = fabs(x - S[i]) / T; if (dd < mg) mg = dd; }
    return mg;
}

/* Exact updated sampling over float biases (Fig. 6(b)): the CTPS of
 * the positive-bias, untaken candidates (ascending), summed left to right in
 * fp64, searched at x = r(U) * T'.  *mg = min(*mg, margin of that draw). */
static int64_t updated_pick_float(const float *b, int64_t n, const int64_t *picks, int64_t taken, uint64_t U,
                                  double *mg)
{
    int64_t nsv = 0;
    int64_t *sv = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    float *b2 = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; i++)
        if (b[i] > 0.0f && !in_list(picks, taken, i)) { sv[nsv] = i; b2[nsv] = b[i]; nsv++; }
    double *S2 = (double *)malloc(sizeof(double) * (size_t)(nsv + 1));
    S2[0] = 0.0;
    for (int64_t i = 0; i < nsv; i++) S2[i + 1] = S2[i] + (double)b2[i];
    double x = unit_r(U) * S2[nsv];
    int64_t q = its_float(S2, b2, nsv, x);
    double m = margin_float(S2, nsv, x, S2[nsv]);
    if (m < *mg) *mg = m;
    int64_t s = sv[q];
    free(S2); free(b2); free(sv);
    return s;
}

/*
 * select_wor over fp32 biases (R28 float path of the box steps):
 * S[0] = 0, S[i+1] = S[i] + (double)b[i] left to right, T = S[n]; every draw is
 * x = r(U) * M for the space size M it draws over.
 *   (1)(2) s = its(S, r(U(j,a)) * T); accept if not taken
 *   (3)    fresh x' = r(U(j,a+1)) * (T - b[s]) over the space without the taken
 *          region [S[s], S[s] + b[s]) (R1; b[s] the region's bias, in fp64)
 *   (4)(5) y = x' if x' < S[s] else x' + b[s]; s = its(S, y); accept if not
 *          taken, else back to (1)
 *   after a_max attempts: exact updated sampling with U(j, a_max) (R2).
 * If k >= #positive-bias candidates: all of them, ascending (R8).
 * *margin (nullable) = the minimum boundary margin over every draw searched
 * (R28: a GPU pick may differ from this one only if it is <= 1e-6).
 */
ORACLE_EXPORT int64_t oracle_select_wor_float(const float *b, int64_t n, int64_t k,
                                              uint64_t seed, uint32_t inst, uint32_t t, uint32_t slot,
                                              int32_t a_max, int64_t *picks, double *margin)
{
    double mg = 1.0;
    int64_t npos = 0;
    for (int64_t i = 0; i < n; i++) if (b[i] > 0.0f) npos++;
    if (margin) *margin = 1.0;
    if (k <= 0 || npos == 0) return 0;
    if (k >= npos) {
        int64_t c = 0;
        for (int64_t i = 0; i < n; i++) if (b[i] > 0.0f) picks[c++] = i;
        return c;
    }
    double *S = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    S[0] = 0.0;
    for (int64_t i = 0; i < n; i++) S[i + 1] = S[i] + (double)b[i];
    double T = S[n];
    int64_t taken = 0;
    for (int64_t j = 0; j < k; j++) {
        uint32_t a = 0;
        int64_t s;
        for (;;) {
            double x = unit_r(draw_u64(seed, inst, t, slot, word3_of(P_EDGE, (uint32_t)j, a), 0)) * T;
            a += 1;
            s = its_float(S, b, n, x);
            double m = margin_float(S, n, x, T);
            if (m < mg) mg = m;
            if (!in_list(picks, taken, s)) break;
            double L = S[s], d = (double)b[s];
            double x2 = unit_r(draw_u64(seed, inst, t, slot, word3_of(P_EDGE, (uint32_t)j, a), 0)) * (T - d);
            a += 1;
            double y = (x2 < L) ? x2 : x2 + d;
            s = its_float(S, b, n, y);
            m = margin_float(S, n, y, T);
            if (m < mg) mg = m;
            if (!in_list(picks, taken, s)) break;
            if ((int32_t)a >= a_max) {
                s = updated_pick_float(b, n, picks, taken,
                                       draw_u64(seed, inst, t, slot, word3_of(P_EDGE, (uint32_t)j, (uint32_t)a_max), 0),
                                       &mg);
                break;
            }
        }
        picks[taken++] = s;
    }
    free(S);
    if (margin) *margin = mg;
    return taken;
}

/* One step of the edge-weight walk at v (biased DeepWalk with EdgeBias = w(e),
 * P:172 with Eq. 3's f(e)): b[i] = w[row_ptr[v] + i], oracle_select_float with
 * U(i, t, 0, EDGE).  Returns the next vertex, or 0xFFFFFFFF if the row's weights
 * sum to 0 (R20).  *margin (nullable) = that draw's boundary margin (R28). */
ORACLE_EXPORT uint32_t oracle_weight_walk_step(const int64_t *row_ptr, const uint32_t *col, const float *w,
                                               int64_t V, uint32_t v, uint32_t inst, uint32_t t, uint64_t rng_seed,
                                               double *margin)
{
    (void)V;
    int64_t n = row_ptr[v + 1] - row_ptr[v];
    if (margin) *margin = 1.0;
    if (n == 0) return 0xFFFFFFFFu;
    uint64_t U = draw_u64(rng_seed, inst, t, 0, word3_of(P_EDGE, 0, 0), 0);
    int64_t s = oracle_select_float(w + row_ptr[v], n, U, margin);
    return s < 0 ? 0xFFFFFFFFu : col[row_ptr[v] + s];
}

ORACLE_EXPORT void oracle_weight_walk(const int64_t *row_ptr, const uint32_t *col, const float *w, int64_t V,
                                      int32_t length, uint32_t s0, uint32_t inst, uint64_t rng_seed,
                                      uint32_t *path, double *margins)
{
    path[0] = s0;
    for (int32_t t = 0; t < length; t++) {
        uint32_t v = path[t];
        double mg = 1.0;
        path[t + 1] = (v == 0xFFFFFFFFu) ? 0xFFFFFFFFu
            : oracle_weight_walk_step(row_ptr, col, w, V, v, inst, (uint32_t)t, rng_seed, &mg);
        if (margins) margins[t] = mg;
    }
}

/* node2vec integer scale (R16): smallest m in [1, 2^16] with m/p and m/q
 * integers in [1, 2^32); 0 if none (then the float path applies). */
ORACLE_EXPORT uint32_t oracle_n2v_scale(double p, double q)
{
    for (uint32_t m = 1; m <= 65536u; m++) {
        double a = (double)m / p, c = (double)m / q;
        if (a == floor(a) && c == floor(c) && a >= 1.0 && c >= 1.0 && a < 4294967296.0 && c < 4294967296.0)
            return m;
    }
    return 0;
}

static int cmp_u32(const void *a, const void *b)
{
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return (x > y) - (x < y);
}

/* u in N(prev): rows are sorted ascending (graph invariant), so the C library
 * bsearch is a faithful membership test. */
static int sorted_contains(const uint32_t *a, int64_t n, uint32_t x)
{
    return n > 0 && bsearch(&x, a, (size_t)n, sizeof(uint32_t), cmp_u32) != NULL;
}

/*
 * One node2vec step at v having come from prev (Grover & Leskovec
 * alpha, R16): alpha = 1/p if u == prev, 1 if u in N(prev), 1/q otherwise.
 * Integer path (m = oracle_n2v_scale(p,q) > 0): b = m*alpha in u32, exact.
 * Float path: b = (float)alpha, S summed left to right in double, r =
 * (U >> 11) * 2^-53, x = r * T, s = max{i < n : S[i] <= x}; *margin receives
 * min_{0<i<n} |x - S[i]| / T (the checker's boundary rule, R28).
 * prev == 0xFFFFFFFF means step 0: uniform (R16).
 */
ORACLE_EXPORT uint32_t oracle_node2vec_step(const int64_t *row_ptr, const uint32_t *col, int64_t V,
                                            double p, double q, uint32_t prev, uint32_t v,
                                            uint32_t inst, uint32_t t, uint64_t rng_seed, double *margin)
{
    csr_t g = { row_ptr, col, V };
    int64_t n = deg_of(&g, v);
    const uint32_t *pool = col + row_ptr[v];
    if (margin) *margin = 1.0;
    if (n == 0) return 0xFFFFFFFFu;
    uint64_t U = draw_u64(rng_seed, inst, t, 0, word3_of(P_EDGE, 0, 0), 0);
    if (prev == 0xFFFFFFFFu)
        return pool[oracle_below(U, (uint64_t)n)];
    const uint32_t *np_ = col + row_ptr[prev];
    int64_t nprev = deg_of(&g, prev);
    static double memo_p = -1.0, memo_q = -1.0;   /* single-threaded: memoise the scale */
    static uint32_t memo_m = 0;
    if (p != memo_p || q != memo_q) { memo_m = oracle_n2v_scale(p, q); memo_p = p; memo_q = q; }
    uint32_t m = memo_m;
    if (m > 0) {
        uint32_t wp = (uint32_t)((double)m / p), w1 = m, wq = (uint32_t)((double)m / q);
        uint64_t *S = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(n + 1));
        S[0] = 0;
        for (int64_t i = 0; i < n; i++) {
            uint32_t u = pool[i];
            uint32_t b = (u == prev) ? wp : (sorted_contains(np_, nprev, u) ? w1 : wq);
            S[i + 1] = S[i] + b;
        }
        uint32_t r = pool[oracle_its(S, n, oracle_below(U, S[n]))];
        free(S);
        return r;
    }
    float fp = (float)(1.0 / p), f1 = 1.0f, fq = (float)(1.0 / q);
    float *b = (float *)malloc(sizeof(float) * (size_t)n);
    for (int64_t i = 0; i < n; i++) {
        uint32_t u = pool[i];
        b[i] = (u == prev) ? fp : (sorted_contains(np_, nprev, u) ? f1 : fq);
    }
    int64_t s = oracle_select_float(b, n, U, margin);
    free(b);
    return pool[s];
}

/* node2vec walk: path[0] = s0; step 0 uniform; then oracle_node2vec_step.
 * margins[t] (nullable) = boundary margin of step t (float path only). */
ORACLE_EXPORT void oracle_node2vec(const int64_t *row_ptr, const uint32_t *col, int64_t V,
                                   double p, double q, int32_t length, uint32_t s0, uint32_t inst,
                                   uint64_t rng_seed, uint32_t *path, double *margins)
{
    path[0] = s0;
    for (int32_t t = 0; t < length; t++) {
        uint32_t v = path[t];
        uint32_t prev = (t == 0) ? 0xFFFFFFFFu : path[t - 1];
        double mg = 1.0;
        path[t + 1] = (v == 0xFFFFFFFFu) ? 0xFFFFFFFFu
            : oracle_node2vec_step(row_ptr, col, V, p, q, prev, v, inst, (uint32_t)t, rng_seed, &mg);
        if (margins) margins[t] = mg;
    }
}

/*
 * Weighted node2vec step (the bias "depends upon the edge weight and its distance
 * from the vertex explored at preceding step"; Grover & Leskovec: alpha(prev, u) * w(v, u);
 * reading R33): b_i = fp32(alpha_i) * w[row_ptr[v] + i] as one fp32 multiply, alpha as in
 * R16 ((float)(1/p) if u == prev, 1 if u in N(prev), (float)(1/q) otherwise), then the float
 * path oracle_select_float (R28).  prev == 0xFFFFFFFF (step 0): b_i = w_i (the weighted
 * walk's step).  *margin (nullable) = the draw's boundary margin.
 */
ORACLE_EXPORT uint32_t oracle_node2vec_w_step(const int64_t *row_ptr, const uint32_t *col, const float *w,
                                              int64_t V, double p, double q, uint32_t prev, uint32_t v,
                                              uint32_t inst, uint32_t t, uint64_t rng_seed, double *margin)
{
    csr_t g = { row_ptr, col, V };
    int64_t n = deg_of(&g, v);
    const uint32_t *pool = col + row_ptr[v];
    const float *wv = w + row_ptr[v];
    if (margin) *margin = 1.0;
    if (n == 0) return 0xFFFFFFFFu;
    uint64_t U = draw_u64(rng_seed, inst, t, 0, word3_of(P_EDGE, 0, 0), 0);
    float fp = (float)(1.0 / p), f1 = 1.0f, fq = (float)(1.0 / q);
    float *b = (float *)malloc(sizeof(float) * (size_t)n);
    const uint32_t *np_ = (prev == 0xFFFFFFFFu) ? NULL : col + row_ptr[prev];
    int64_t nprev = (prev == 0xFFFFFFFFu) ? 0 : deg_of(&g, prev);
    for (int64_t i = 0; i < n; i++) {
        uint32_t u = pool[i];
        float a = (prev == 0xFFFFFFFFu) ? 1.0f : (u == prev ? fp : (sorted_contains(np_, nprev, u) ? f1 : fq));
        b[i] = a * wv[i];
    }
    int64_t s = oracle_select_float(b, n, U, margin);
    free(b);
    return s < 0 ? 0xFFFFFFFFu : pool[s];
}

ORACLE_EXPORT void oracle_node2vec_w(const int64_t *row_ptr, const uint32_t *col, const float *w, int64_t V,
                                     double p, double q, int32_t length, uint32_t s0, uint32_t inst,
                                     uint64_t rng_seed, uint32_t *path, double *margins)
{
    path[0] = s0;
    for (int32_t t = 0; t < length; t++) {
        uint32_t v = path[t];
        uint32_t prev = (t == 0) ? 0xFFFFFFFFu : path[t - 1];
        double mg = 1.0;
        path[t + 1] = (v == 0xFFFFFFFFu) ? 0xFFFFFFFFu
            : oracle_node2vec_w_step(row_ptr, col, w, V, p, q, prev, v, inst, (uint32_t)t, rng_seed, &mg);
        if (margins) margins[t] = mg;
    }
}

/*
 * Multi-dimensional random walk (frontier sampling; Fig. 4):
 * pool = seeds[0..m) in slot order (R18); per step t: VertexBias = degree,
 * slot = its(S(pool), below(U(i,t,0,VERTEX), T)); v = pool[slot];
 * EdgeBias = 1 -> u = N(v)[below(U(i,t,0,EDGE), deg v)] (closed form of ITS
 * with unit biases); Update: pool[slot] = u (in-place, R18).
 * edges[2t] = v, edges[2t+1] = u.  A pool of total degree 0 ends the walk (pad).
 */
ORACLE_EXPORT void oracle_mdrw(const int64_t *row_ptr, const uint32_t *col, int64_t V,
                               const uint32_t *seeds, int32_t m, int32_t steps, uint32_t inst, uint64_t rng_seed,
                               uint32_t *edges)
{
    csr_t g = { row_ptr, col, V };
    uint32_t *pool = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)m);
    uint32_t *b = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)m);
    uint64_t *S = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(m + 1));
    memcpy(pool, seeds, sizeof(uint32_t) * (size_t)m);
    for (int32_t t = 0; t < steps; t++) {
        for (int32_t i = 0; i < m; i++) b[i] = (uint32_t)deg_of(&g, pool[i]);
        oracle_prefix(b, m, S);
        if (S[m] == 0) {
            for (int32_t r = t; r < steps; r++) { edges[2 * r] = 0xFFFFFFFFu; edges[2 * r + 1] = 0xFFFFFFFFu; }
            break;
        }
        uint64_t xv = oracle_below(draw_u64(rng_seed, inst, (uint32_t)t, 0, word3_of(P_VERTEX, 0, 0), 0), S[m]);
        int64_t slot = oracle_its(S, m, xv);
        uint32_t v = pool[slot];
        uint64_t xe = oracle_below(draw_u64(rng_seed, inst, (uint32_t)t, 0, word3_of(P_EDGE, 0, 0), 0), (uint64_t)deg_of(&g, v));
        uint32_t u = col[row_ptr[v] + (int64_t)xe];
        edges[2 * t] = v;
        edges[2 * t + 1] = u;
        pool[slot] = u;
    }
    free(S); free(b); free(pool);
}

/* ------------------------------------------------------------------------- */
/* Out-of-memory scheduling facts (§5.2).                         */
/* ------------------------------------------------------------------------- */

/* Equal contiguous vertex ranges, remainder to the lowest partitions (R23):
 * bounds[0..P]. */
ORACLE_EXPORT void oracle_partition_bounds(int64_t V, int32_t P, int64_t *bounds)
{
    int64_t base = V / P, rem = V % P, acc = 0;
    bounds[0] = 0;
    for (int32_t p = 0; p < P; p++) { acc += base + (p < rem ? 1 : 0); bounds[p + 1] = acc; }
}

/* Active-vertex count per partition for a frontier. */
ORACLE_EXPORT void oracle_active_counts(const int64_t *bounds, int32_t P, const uint32_t *frontier, int64_t n,
                                        int64_t *counts)
{
    for (int32_t p = 0; p < P; p++) counts[p] = 0;
    for (int64_t i = 0; i < n; i++)
        for (int32_t p = 0; p < P; p++)
            if ((int64_t)frontier[i] >= bounds[p] && (int64_t)frontier[i] < bounds[p + 1]) { counts[p]++; break; }
}
