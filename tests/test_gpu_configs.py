"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Each test builds the config's full synthetic graph on the GPU, runs the whole
workload through the C ABI exactly as bench.py does (all instances in one
call), and compares a deterministic sample of instances / walkers with the
oracle element by element (integer biases: bit-exact).  Invariants that hold
at any size are checked on 100 % of the output.
"""
import gc
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import CONFIGS, instance_seeds, mdrw_seeds, nonisolated_vertices, rmat_csr
from tests._parity import DEV, u32

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

# Philox seed of the runs (CSAW_TEST_SEED overrides: the same checks under other random streams)
SEED = int(os.environ.get("CSAW_TEST_SEED", "1"))


def build(cfg, ctps_cache=False, node2vec_tri=False):
    g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=DEV)
    G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, ctps_cache=ctps_cache, node2vec_tri=node2vec_tri)
    og = O.Graph(g.row_ptr.cpu().numpy(), g.col_idx.cpu().numpy().view(np.uint32))
    return g, G, og


def release(*objs):
    for o in objs:
        if isinstance(o, cs.Graph):
            o.close()
    gc.collect()
    torch.cuda.empty_cache()


def sample_ids(n, k, salt=0):
    """Deterministic spread of k ids in [0, n) incl. the first and last."""
    if n <= k:
        return list(range(n))
    ids = set(np.linspace(0, n - 1, k - 8).astype(np.int64).tolist())
    rng = np.random.default_rng(1234 + salt)
    ids |= set(rng.integers(0, n, 8).tolist())
    return sorted(ids)


def check_edges_exist(og, src, dst):
    """every sampled (src, dst) is a CSR edge (vectorised binary search per row)."""
    rp = og.row_ptr
    for s, d in zip(src[:: max(1, len(src) // 200000)], dst[:: max(1, len(dst) // 200000)]):
        row = og.col[rp[s]:rp[s + 1]]
        i = np.searchsorted(row, d)
        assert i < row.size and row[i] == d


@pytest.mark.parametrize("cached", [False, True])
def test_cfg2_degree_walk_full(cached):
    """cached=True is the bench's launch: CTPS cache + narrow walk index (k_walk_wix)."""
    cfg = CONFIGS["cfg2"]
    g, G, og = build(cfg, ctps_cache=cached)
    assert G.info()["walk_index_leaf"] == (128 if cached else 0)
    seeds = instance_seeds(g, cfg.n_instances).to(DEV)
    path = u32(cs.csaw_walk(G, "degree", seeds, cfg.length, rng_seed=SEED))
    assert path.shape == (cfg.n_instances, cfg.length + 1)
    assert (path != cs.NONE).all()                       # symmetric graph, non-isolated seeds: exact length
    sv = u32(seeds)
    for w in sample_ids(cfg.n_instances, 24):
        ref = O.walk(og, O.KIND_DEGREE, cfg.length, int(sv[w]), w, SEED)
        assert np.array_equal(path[w], ref), f"walker {w}"
    # 100 % invariant: consecutive path vertices are adjacent
    check_edges_exist(og, path[:, :-1].ravel(), path[:, 1:].ravel())
    release(G)


@pytest.mark.parametrize("cached", [False, True])
def test_cfg3_node2vec_full(cached):
    """cached=True is the bench's launch: per-edge triangle counts + partial scans (k_node2vec_tri)."""
    cfg = CONFIGS["cfg3"]
    g, G, og = build(cfg, node2vec_tri=cached)
    assert G.info()["node2vec_tri"] == (1 if cached else 0)
    seeds = nonisolated_vertices(g).to(torch.int32).to(DEV)
    n = seeds.numel()
    path = u32(cs.csaw_walk(G, cs.make_bias("node2vec", p=cfg.p, q=cfg.q), seeds, cfg.length, rng_seed=SEED))
    assert path.shape == (n, cfg.length + 1) and (path != cs.NONE).all()
    sv = u32(seeds)
    for w in sample_ids(n, 40):
        ref = O.node2vec(og, cfg.p, cfg.q, cfg.length, int(sv[w]), w, SEED)
        assert np.array_equal(path[w], ref), f"walker {w}"
    check_edges_exist(og, path[:, :-1].ravel(), path[:, 1:].ravel())
    release(G)


def _check_sampling(cfg, g, G, og, workload, k_sample=160):
    seeds = instance_seeds(g, cfg.n_instances).to(DEV)
    bias = cs.make_bias(cfg.bias, pf=cfg.pf)
    offs, src, dst, dep = cs.csaw_sample(G, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth, rng_seed=SEED)
    offs = offs.cpu().numpy().astype(np.int64)
    src, dst, dep = u32(src), u32(dst), dep.cpu().numpy()
    sv = u32(seeds)
    for i in sample_ids(cfg.n_instances, k_sample):
        if workload == "layer":
            es, ed, ee = O.layer_sample(og, list(cfg.fanout), cfg.depth, int(sv[i]), i, SEED)
        else:
            es, ed, ee = O.neighbor_sample(og, O.KIND_FF, [], cfg.depth, int(sv[i]), i, SEED, cfg.pf)
        a, b = offs[i], offs[i + 1]
        assert np.array_equal(src[a:b], es) and np.array_equal(dst[a:b], ed) and np.array_equal(dep[a:b], ee), i
    check_edges_exist(og, src, dst)
    assert (dep >= 1).all() and (dep <= cfg.depth).all()
    return offs


def test_cfg4_layer_and_forest_fire_full():
    cfg = CONFIGS["cfg4_layer"]
    g, G, og = build(cfg)
    offs = _check_sampling(cfg, g, G, og, "layer")
    # layer: exactly min(fanout, pool) per level -> 4 edges per instance when pools are large
    assert np.median(np.diff(offs)) == 4
    _check_sampling(CONFIGS["cfg4_ff"], g, G, og, "forest_fire")
    release(G)


def test_cfg5_mdrw_in_memory_full():
    cfg = CONFIGS["cfg5"]
    g, G, og = build(cfg)
    seeds = mdrw_seeds(g, cfg.n_instances, cfg.pool_size).to(DEV)
    edges = u32(cs.csaw_walk(G, cs.make_bias("mdrw"), seeds, cfg.length, rng_seed=SEED))
    assert edges.shape == (cfg.n_instances, cfg.length, 2) and (edges != cs.NONE).all()
    sv = u32(seeds)
    for i in sample_ids(cfg.n_instances, 16):
        ref = O.mdrw(og, sv[i], cfg.length, i, SEED)
        assert np.array_equal(edges[i], ref), f"instance {i}"
    check_edges_exist(og, edges[:, :, 0].ravel(), edges[:, :, 1].ravel())
    release(G)
    # the config's out-of-memory launch (8 GB budget), zero-copy mode with the resident
    # col_idx prefix: identical to the in-memory edges on 100 % of the output
    Gz = cs.csaw_graph_create(g.row_ptr.cpu(), g.col_idx.cpu(), device=0, budget_bytes=cfg.oom_budget_bytes,
                              num_partitions=cfg.oom_partitions, max_resident=1, zerocopy=True)
    assert Gz.info()["device_bytes"] <= cfg.oom_budget_bytes
    ez = u32(cs.csaw_walk(Gz, cs.make_bias("mdrw"), seeds, cfg.length, rng_seed=SEED))
    assert np.array_equal(ez, edges)
    release(Gz)
