"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Each test builds the config's full synthetic graph on the GPU, runs the whole
workload through the C ABI exactly as bench.py does (all instances in one call),
and compares with the oracle element by element (integer biases: bit-exact) at
the coverage SURVEY.md §8(d) d.4 plans:

  cfg2  all 4,000 walkers                      (cache + walk index, and the scan paths: deg
                                               gathers and the streamed materialised bias);
        cfg2_weight: all 4,000 edge-weight walkers (float path, 1e-6 boundary rule)
  cfg3  every 64th walker (~29.5K of ~1.9M)    (intersection index = the bench's launch);
        the index, triangle-count and full-merge kernels are also compared with each
        other on 100 % of the walkers
  cfg4  all 8,192 instances, layer and forest fire
  cfg5  all 4,000 MDRW instances in memory; the 8 GB OOM launches (zero-copy and the
        paper's partition scheduling) equal to the in-memory output on 100 %
  cfg5_ns all 8,192 instances in memory; OOM partition scheduling / zero-copy equal

each for the three rng seeds of §8(d) d.2 (CSAW_TEST_SEEDS overrides, e.g. "1").
The oracle is fanned out over the host cores (instances are independent).
Invariants that hold at any size are checked on 100 % of the output.
"""
import gc
import os
import time

import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import CONFIGS, instance_seeds, mdrw_seeds, nonisolated_vertices, rmat_csr
from tests._parity import DEV, u32

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SEEDS = [int(s) for s in os.environ.get("CSAW_TEST_SEEDS", os.environ.get("CSAW_TEST_SEED", "1,2,3")).split(",")]


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


def release(*objs):
    for o in objs:
        if isinstance(o, cs.Graph):
            o.close()
    gc.collect()
    torch.cuda.empty_cache()


def first_mismatch(got, ref):
    """index of the first differing row (None if equal)"""
    bad = np.nonzero((got != ref).reshape(got.shape[0], -1).any(axis=1))[0]
    return None if bad.size == 0 else int(bad[0])


def check_edges_exist(og, src, dst):
    """every (src, dst) is a CSR edge: vectorised binary search inside each src row"""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.uint32)
    lo, hi = og.row_ptr[src], og.row_ptr[src + 1]
    assert (hi > lo).all()
    # lower bound of dst within col[lo:hi), all rows at once
    while True:
        act = lo < hi
        if not act.any():
            break
        mid = (lo + hi) // 2
        less = og.col[np.where(act, mid, 0)] < dst
        lo = np.where(act & less, mid + 1, lo)
        hi = np.where(act & ~less, mid, hi)
    assert (lo < og.row_ptr[src + 1]).all() and (og.col[np.minimum(lo, og.col.size - 1)] == dst).all()


def flat_sampling(offs, src, dst, dep, ids):
    return [(src[offs[i]:offs[i + 1]], dst[offs[i]:offs[i + 1]], dep[offs[i]:offs[i + 1]]) for i in ids]


def compare_sampling(got, ref, what):
    for i, ((a, b, c), (x, y, z)) in enumerate(zip(got, ref)):
        assert np.array_equal(a, x) and np.array_equal(b, y) and np.array_equal(c, z), f"{what}: instance {i}"


def run_sample(G, bias, seeds, cfg, seed):
    offs, src, dst, dep = cs.csaw_sample(G, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth, rng_seed=seed)
    torch.cuda.synchronize()
    return offs.cpu().numpy().astype(np.int64), u32(src), u32(dst), dep.cpu().numpy()


# ------------------------------------------------------------------ cfg2
def test_cfg2_degree_walk_full():
    cfg = CONFIGS["cfg2"]
    g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=DEV)
    og = O.Graph.from_torch(g)
    seeds = instance_seeds(g, cfg.n_instances).to(DEV)
    sv = u32(seeds)
    Gc = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, ctps_cache=True)     # the bench's launch
    Gs = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0)                      # per-step scans (the ★ path)
    Ge = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, edge_bias=True)      # per-step scans of the streamed bias
    Gb = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, ctps_cache=True, walk_buckets=True)   # k_walk_gb
    assert Gc.info()["walk_index_leaf"] == 128 and Gs.info()["ctps_cache"] == 0 and Ge.info()["edge_bias"] == 1
    assert Gb.info()["walk_buckets"] == 1
    for seed in SEEDS:
        pc = u32(cs.csaw_walk(Gc, "degree", seeds, cfg.length, rng_seed=seed))
        pb = u32(cs.csaw_walk(Gb, "degree", seeds, cfg.length, rng_seed=seed))
        assert first_mismatch(pb, pc) is None, f"seed {seed}: bucket vs head walker {first_mismatch(pb, pc)}"
        ps = u32(cs.csaw_walk(Gs, "degree", seeds, cfg.length, rng_seed=seed))
        pe = u32(cs.csaw_walk(Ge, "degree", seeds, cfg.length, rng_seed=seed))
        assert first_mismatch(pe, ps) is None, f"seed {seed}: stream vs gather walker {first_mismatch(pe, ps)}"
        t0 = time.time()
        ref = np.stack(O.parallel_run(og, "walk", sv, 0, seed, kind=O.KIND_DEGREE, length=cfg.length))
        log(f"cfg2 seed {seed}: oracle over all {len(sv)} walkers in {time.time() - t0:.1f} s")
        assert pc.shape == ref.shape == (cfg.n_instances, cfg.length + 1)
        assert first_mismatch(pc, ref) is None, f"seed {seed}: cached walker {first_mismatch(pc, ref)}"
        assert first_mismatch(ps, ref) is None, f"seed {seed}: scan walker {first_mismatch(ps, ref)}"
        assert (pc != cs.NONE).all()          # symmetric graph, non-isolated seeds: exact length
        check_edges_exist(og, pc[:, :-1].ravel(), pc[:, 1:].ravel())
    release(Gc, Gs, Ge, Gb)


def test_cfg2_weight_walk_full():
    """The float path (R28/R32) at config-2 scale: all 4,000 walkers of the edge-weight walk vs the
    oracle; a walk may leave the oracle's only at a step whose draw lies within 1e-6 of a CTPS
    boundary (the oracle reports the margin of every step)."""
    from synth import edge_weights
    cfg = CONFIGS["cfg2_weight"]
    g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=DEV)
    w = edge_weights(g, cfg.graph_seed)
    og = O.Graph.from_torch(g, w)
    seeds = instance_seeds(g, cfg.n_instances).to(DEV)
    sv = u32(seeds)
    G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, weights=w)                       # per-step scans
    Gb = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, weights=w, walk_buckets=True)   # the bench's launch
    assert Gb.info()["walk_buckets"] & 2
    for seed in SEEDS:
        pw = u32(cs.csaw_walk(G, "weight", seeds, cfg.length, rng_seed=seed))
        pb = u32(cs.csaw_walk(Gb, "weight", seeds, cfg.length, rng_seed=seed))
        t0 = time.time()
        ref = O.parallel_run(og, "weight_walk", sv, 0, seed, length=cfg.length)
        log(f"cfg2_weight seed {seed}: oracle over all {len(sv)} walkers in {time.time() - t0:.1f} s")
        excused = 0
        for i, (rp, mg) in enumerate(ref):
            if not np.array_equal(pw[i], rp):
                t = int(np.argmax(pw[i] != rp)) - 1     # the step whose pick differs
                assert mg[t] <= 1e-6, f"seed {seed}: walker {i} step {t} margin {mg[t]}"
                excused += 1
        assert excused <= 4, excused
        # the weighted buckets sum rows left to right like the oracle: every walk is the oracle's
        bad = [i for i, (rp, _) in enumerate(ref) if not np.array_equal(pb[i], rp)]
        assert not bad, f"seed {seed}: bucketed weighted walkers {bad[:5]} differ from the oracle"
        check_edges_exist(og, pw[:, :-1].ravel(), pw[:, 1:].ravel())
    release(G, Gb)


# ------------------------------------------------------------------ cfg3
def test_cfg3_node2vec_full():
    cfg = CONFIGS["cfg3"]
    g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=DEV)
    og = O.Graph.from_torch(g)
    seeds = nonisolated_vertices(g).to(torch.int32).to(DEV)
    n = seeds.numel()
    sv = u32(seeds)
    ids = np.arange(0, n, 64)
    Gx = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, node2vec_index=True)  # the bench's launch
    Gt = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, node2vec_tri=True)    # triangle counts + scans
    Gm = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0)                       # full merge per step
    assert Gx.info()["node2vec_index"] == 1 and Gt.info()["node2vec_tri"] == 1 and Gm.info()["node2vec_tri"] == 0
    bias = cs.make_bias("node2vec", p=cfg.p, q=cfg.q)
    for seed in SEEDS:
        px = u32(cs.csaw_walk(Gx, bias, seeds, cfg.length, rng_seed=seed))
        pt = u32(cs.csaw_walk(Gt, bias, seeds, cfg.length, rng_seed=seed))
        pm = u32(cs.csaw_walk(Gm, bias, seeds, cfg.length, rng_seed=seed))
        assert px.shape == (n, cfg.length + 1) and (px != cs.NONE).all()
        # three independent kernels (intersection index, triangle counts + partial scans,
        # full CTPS merge) on 100 % of the walkers
        assert first_mismatch(px, pm) is None, f"seed {seed}: index vs merge walker {first_mismatch(px, pm)}"
        assert first_mismatch(pt, pm) is None, f"seed {seed}: tri vs merge walker {first_mismatch(pt, pm)}"
        pt = px
        t0 = time.time()
        ref = np.stack(O.parallel_run(og, "node2vec", sv, 0, seed, ids=ids, p=cfg.p, q=cfg.q, length=cfg.length))
        log(f"cfg3 seed {seed}: oracle over {ids.size} walkers (every 64th of {n}) in {time.time() - t0:.1f} s")
        bad = first_mismatch(pt[ids], ref)
        assert bad is None, f"seed {seed}: walker {int(ids[bad])}"
        check_edges_exist(og, pt[::7, :-1].ravel(), pt[::7, 1:].ravel())
    release(Gx, Gt, Gm)


# ------------------------------------------------------------------ cfg4
def test_cfg4_layer_and_forest_fire_full():
    cl, cf = CONFIGS["cfg4_layer"], CONFIGS["cfg4_ff"]
    g = rmat_csr(cl.graph_vertices, cl.graph_entries, cl.graph_seed, device=DEV)
    og = O.Graph.from_torch(g)
    seeds = instance_seeds(g, cl.n_instances).to(DEV)
    sv = u32(seeds)
    ids = np.arange(cl.n_instances)
    Gc = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, ctps_cache=True)     # the bench's launch
    for seed in SEEDS:
        t0 = time.time()
        ref_l = O.parallel_run(og, "layer", sv, 0, seed, fanout=list(cl.fanout), depth=cl.depth)
        ref_f = O.parallel_run(og, "forest_fire", sv, 0, seed, depth=cf.depth, pf=cf.pf)
        log(f"cfg4 seed {seed}: oracle over all {len(sv)} instances (layer + FF) in {time.time() - t0:.1f} s")
        offs, src, dst, dep = run_sample(Gc, cs.make_bias("layer"), seeds, cl, seed)
        compare_sampling(flat_sampling(offs, src, dst, dep, ids), ref_l, f"layer seed {seed}")
        assert np.median(np.diff(offs)) == 4            # min(fanout, pool) per level
        check_edges_exist(og, src, dst)
        offs, src, dst, dep = run_sample(Gc, cs.make_bias("forest_fire", pf=cf.pf), seeds, cf, seed)
        compare_sampling(flat_sampling(offs, src, dst, dep, ids), ref_f, f"forest fire seed {seed}")
        check_edges_exist(og, src, dst)
        assert (dep >= 1).all() and (dep <= cf.depth).all()
    release(Gc)
    # the uncached (per-pool scan) launch on one seed: same bytes
    Gs = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0)
    offs, src, dst, dep = run_sample(Gs, cs.make_bias("layer"), seeds, cl, SEEDS[0])
    ref_l = O.parallel_run(og, "layer", sv, 0, SEEDS[0], fanout=list(cl.fanout), depth=cl.depth)
    compare_sampling(flat_sampling(offs, src, dst, dep, ids), ref_l, "layer (scan)")
    release(Gs)


# ------------------------------------------------------------------ cfg5
@pytest.fixture(scope="module")
def cfg5_graph():
    cfg = CONFIGS["cfg5"]
    g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=DEV)
    og = O.Graph.from_torch(g)
    host = (g.row_ptr.cpu(), g.col_idx.cpu())
    yield g, og, host
    del g
    release()


def oom_graph(host, cfg, zerocopy):
    return cs.csaw_graph_create(host[0], host[1], device=0, budget_bytes=cfg.oom_budget_bytes,
                                num_partitions=cfg.oom_partitions,
                                max_resident=1 if zerocopy else cfg.oom_resident,
                                num_streams=cfg.oom_resident, zerocopy=zerocopy)


def test_cfg5_mdrw_full(cfg5_graph):
    cfg = CONFIGS["cfg5"]
    g, og, host = cfg5_graph
    seeds = mdrw_seeds(g, cfg.n_instances, cfg.pool_size).to(DEV)
    sv = u32(seeds)
    Gm = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, next_record=True)   # in-memory bench launch
    Gp = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0)                     # plain in-memory
    Gn = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, next_meta=True)     # 8 B metadata + col
    bias = cs.make_bias("mdrw")
    inmem = {}
    for seed in SEEDS:
        em = u32(cs.csaw_walk(Gm, bias, seeds, cfg.length, rng_seed=seed))
        ep = u32(cs.csaw_walk(Gp, bias, seeds, cfg.length, rng_seed=seed))
        t0 = time.time()
        ref = np.stack(O.parallel_run(og, "mdrw", sv, 0, seed, length=cfg.length))
        log(f"cfg5 seed {seed}: oracle over all {len(sv)} MDRW instances in {time.time() - t0:.1f} s")
        assert em.shape == ref.shape == (cfg.n_instances, cfg.length, 2) and (em != cs.NONE).all()
        assert first_mismatch(em, ref) is None, f"seed {seed}: instance {first_mismatch(em, ref)}"
        assert first_mismatch(ep, ref) is None, f"seed {seed}: plain instance {first_mismatch(ep, ref)}"
        check_edges_exist(og, em[:, :, 0].ravel(), em[:, :, 1].ravel())
        if seed == SEEDS[0]:
            en = u32(cs.csaw_walk(Gn, bias, seeds, cfg.length, rng_seed=seed))
            assert first_mismatch(en, em) is None, "next_meta vs next_record"
        inmem[seed] = em
    release(Gm, Gp, Gn)
    # the config's out-of-memory launches under the 8 GB budget: identical on 100 %
    Gz = oom_graph(host, cfg, zerocopy=True)
    assert Gz.info()["oom_mode"] == 1 and Gz.info()["device_bytes"] <= cfg.oom_budget_bytes
    for seed in SEEDS:
        ez = u32(cs.csaw_walk(Gz, bias, seeds, cfg.length, rng_seed=seed))
        assert first_mismatch(ez, inmem[seed]) is None, f"zero-copy seed {seed}"
    release(Gz)
    Go = oom_graph(host, cfg, zerocopy=False)                  # the paper's partition scheduling (§5)
    assert Go.info()["oom_mode"] == 1 and Go.info()["device_bytes"] <= cfg.oom_budget_bytes
    t0 = time.time()
    eo = u32(cs.csaw_walk(Go, bias, seeds, cfg.length, rng_seed=SEEDS[0]))
    st = cs.csaw_stats(Go)
    log(f"cfg5 partition-scheduled OOM MDRW: {time.time() - t0:.1f} s, {st['partition_loads']} partition loads")
    assert st["partition_loads"] > cfg.oom_resident
    assert first_mismatch(eo, inmem[SEEDS[0]]) is None, "partition-scheduled OOM MDRW"
    release(Go)


def test_cfg5_ns_full(cfg5_graph):
    cfg = CONFIGS["cfg5_ns"]
    g, og, host = cfg5_graph
    seeds = instance_seeds(g, cfg.n_instances).to(DEV)
    sv = u32(seeds)
    ids = np.arange(cfg.n_instances)
    bias = cs.make_bias("degree")
    Gm = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0)
    inmem = {}
    for seed in SEEDS:
        r = run_sample(Gm, bias, seeds, cfg, seed)
        t0 = time.time()
        ref = O.parallel_run(og, "degree", sv, 0, seed, fanout=list(cfg.fanout), depth=cfg.depth)
        log(f"cfg5_ns seed {seed}: oracle over all {len(sv)} instances in {time.time() - t0:.1f} s")
        compare_sampling(flat_sampling(*r, ids), ref, f"cfg5_ns in memory seed {seed}")
        check_edges_exist(og, r[1], r[2])
        inmem[seed] = r
    release(Gm)
    for zc in (False, True):
        Go = oom_graph(host, cfg, zerocopy=zc)
        assert Go.info()["oom_mode"] == 1 and Go.info()["device_bytes"] <= cfg.oom_budget_bytes
        for seed in SEEDS:
            r = run_sample(Go, bias, seeds, cfg, seed)
            for a, b in zip(r, inmem[seed]):
                assert np.array_equal(a, b), f"cfg5_ns OOM ({'zero-copy' if zc else 'partitions'}) seed {seed}"
            if not zc:
                assert cs.csaw_stats(Go)["partition_loads"] >= cfg.oom_partitions
        release(Go)
