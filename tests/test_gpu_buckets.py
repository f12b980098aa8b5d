"""Degree walks over the bucketed walk index (CSAW_GRAPH_WALK_BUCKETS, k_walk_gb): one 128 B
bucket line per step, a link into the CTPS cache when more than 8 regions meet a bucket.  Must be
bit-identical to the oracle's degree walk (same integer S, same draw, same region) and to the
vertex-head kernel, on R-MAT graphs, on the hub graph, and on a graph whose buckets overflow."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import instance_seeds, rmat_csr
from tests._golden import gtoy
from tests._parity import DEV, check_walk, u32
from tests.test_gpu_parity import hub_csr

pytestmark = pytest.mark.gpu


def graphs(rp, col):
    rpt = torch.as_tensor(np.asarray(rp, dtype=np.int64))
    ct = torch.as_tensor(np.asarray(col).astype(np.uint32).view(np.int32))
    Gb = cs.csaw_graph_create(rpt.to(DEV), ct.to(DEV), ctps_cache=True, walk_buckets=True)
    Gh = cs.csaw_graph_create(rpt.to(DEV), ct.to(DEV), ctps_cache=True)   # vertex heads (k_walk_head)
    return Gb, Gh, O.Graph(rpt.numpy(), ct.numpy().view(np.uint32))


def skew_csr():
    """Vertex 0 adjacent to hubs 1..4 (degree ~50,000 each) and to 2,000 leaves: row 0's
    mean region width is ~100, so its 2,000 unit regions crowd ~64 to a bucket (links)."""
    edges = set()
    leaf = 5
    for h in range(1, 5):
        edges.add((0, h))
        for _ in range(50_000):
            edges.add((h, leaf))
            leaf += 1
    for _ in range(2_000):
        edges.add((0, leaf))
        leaf += 1
    V = leaf
    e = np.array(sorted(edges), dtype=np.int64)
    src = np.concatenate([e[:, 0], e[:, 1]])
    dst = np.concatenate([e[:, 1], e[:, 0]])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    rp = np.zeros(V + 1, np.int64)
    np.add.at(rp, src + 1, 1)
    return np.cumsum(rp), dst.astype(np.uint32)


def test_buckets_gtoy():
    rp, col = gtoy()
    Gb, Gh, og = graphs(rp, col)
    assert Gb.info()["walk_buckets"] == 1 and Gh.info()["walk_buckets"] == 0
    seeds = np.arange(len(rp) - 1, dtype=np.uint32)
    check_walk(Gb, og, "degree", seeds, 50, rng_seed=4)
    Gb.close(); Gh.close()


@pytest.mark.parametrize("seed", [1, 2])
def test_buckets_rmat(seed):
    g = rmat_csr(1 << 15, 1 << 19, 7, device=DEV).to("cpu")
    Gb, Gh, og = graphs(g.row_ptr, g.col_idx)
    assert Gb.info()["walk_buckets"] == 1
    seeds = instance_seeds(g, 512, set_id=seed).numpy()
    pb = check_walk(Gb, og, "degree", seeds, 300, rng_seed=seed, walkers=range(0, 512, 4))
    st = cs.csaw_stats(Gb)
    assert st["pools"] > 0
    ph = u32(cs.csaw_walk(Gh, "degree", torch.as_tensor(seeds.view(np.int32)).to(DEV), 300, rng_seed=seed))
    assert np.array_equal(pb, ph)
    Gb.close(); Gh.close()


def test_buckets_hub():
    rp, col = hub_csr()
    Gb, Gh, og = graphs(rp, col)
    seeds = np.array([0, 1, 0, 1, 5, 0, 1, 17, 299_999, 20_001] * 8, dtype=np.uint32)
    check_walk(Gb, og, "degree", seeds, 200, rng_seed=9, walkers=range(10))
    ph = u32(cs.csaw_walk(Gh, "degree", torch.as_tensor(seeds.view(np.int32)).to(DEV), 200, rng_seed=9))
    pb = u32(cs.csaw_walk(Gb, "degree", torch.as_tensor(seeds.view(np.int32)).to(DEV), 200, rng_seed=9))
    assert np.array_equal(pb, ph)
    Gb.close(); Gh.close()


def test_buckets_overflow_links():
    """Buckets met by more than 8 regions continue in the CTPS cache (counted in
    csaw_run_stats.cache_probes); picks stay identical to the oracle and the head kernel."""
    rp, col = skew_csr()
    Gb, Gh, og = graphs(rp, col)
    seeds = np.zeros(2048, dtype=np.uint32)   # every walker starts at row 0 (the crowded buckets)
    seeds[1::2] = 5                           # and at a leaf of hub 1
    st_path = u32(cs.csaw_walk(Gb, "degree", torch.as_tensor(seeds.view(np.int32)).to(DEV), 64, rng_seed=3))
    st = cs.csaw_stats(Gb)
    assert st["cache_probes"] > 0, "no bucket link was taken"
    check_walk(Gb, og, "degree", seeds, 64, rng_seed=3, walkers=range(0, 2048, 16))
    ph = u32(cs.csaw_walk(Gh, "degree", torch.as_tensor(seeds.view(np.int32)).to(DEV), 64, rng_seed=3))
    assert np.array_equal(st_path, ph)
    Gb.close(); Gh.close()


def test_buckets_sharding_and_seeds():
    """instance_base offsets the Philox counters exactly as in the other kernels; a seed >= V
    is OUT_OF_RANGE before any walk kernel."""
    g = rmat_csr(1 << 12, 1 << 16, 3, device=DEV).to("cpu")
    Gb, Gh, og = graphs(g.row_ptr, g.col_idx)
    seeds = instance_seeds(g, 64, set_id=2).numpy()
    check_walk(Gb, og, "degree", seeds, 80, rng_seed=6, instance_base=1000)
    bad = torch.tensor([0, g.row_ptr.numel() + 5], dtype=torch.int32, device=DEV)
    with pytest.raises(cs.CsawError):
        cs.csaw_walk(Gb, "degree", bad, 10, rng_seed=1)
    Gb.close(); Gh.close()


# ------------------------------------------------------------------ edge weights (float path, R28)
def weighted(rp, col, w):
    rpt = torch.as_tensor(np.asarray(rp, dtype=np.int64))
    ct = torch.as_tensor(np.asarray(col).astype(np.uint32).view(np.int32))
    wt = torch.as_tensor(np.asarray(w, dtype=np.float32))
    G = cs.csaw_graph_create(rpt.to(DEV), ct.to(DEV), weights=wt.to(DEV), walk_buckets=True)
    return G, O.Graph(rpt.numpy(), ct.numpy().view(np.uint32), wt.numpy())


def check_weight_exact(G, og, seeds, length, rng_seed, walkers):
    path = u32(cs.csaw_walk(G, "weight", torch.as_tensor(np.asarray(seeds, np.uint32).view(np.int32)).to(DEV),
                            length, rng_seed=rng_seed))
    for i in walkers:
        ref = O.weight_walk(og, length, int(seeds[i]), i, rng_seed)
        if not np.array_equal(path[i], ref):
            t = int(np.argmax(path[i] != ref))
            raise AssertionError(f"walker {i}: first divergence at {t}: gpu {path[i][t]} oracle {ref[t]}")
    return path


@pytest.mark.parametrize("zero_frac", [0.0, 0.2])
def test_weight_buckets_exact(zero_frac):
    """The weighted buckets sum each row left to right in fp64 like the oracle, so weighted
    walks equal the oracle's exactly (no 1e-6 boundary excuse)."""
    from synth import edge_weights
    g = rmat_csr(1 << 15, 1 << 19, 5, device=DEV).to("cpu")
    w = edge_weights(g, 3, zero_frac=zero_frac)
    G, og = weighted(g.row_ptr, g.col_idx, w)
    assert G.info()["walk_buckets"] & 2
    seeds = instance_seeds(g, 512, set_id=3).numpy()
    check_weight_exact(G, og, seeds, 300, 5, range(0, 512, 3))
    G.close()


def test_weight_buckets_links():
    """Row 0: four unit-weight hubs and 2,000 leaves of weight 2^-14 -- 32 leaf regions per
    bucket, so buckets link into the fp64 prefix; picks still equal the oracle's."""
    rp, col = skew_csr()
    src = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    w = np.ones(len(col), np.float32)
    w[(src == 0) & (col >= 5)] = 2.0 ** -14
    w[(col == 0) & (src >= 5)] = 0.5
    G, og = weighted(rp, col, w)
    assert G.info()["walk_buckets"] & 2
    seeds = np.zeros(2048, dtype=np.uint32)
    seeds[1::2] = 5
    check_weight_exact(G, og, seeds, 64, 8, range(0, 2048, 7))
    assert cs.csaw_stats(G)["cache_probes"] > 0, "no weighted bucket link was taken"
    G.close()


def directed_csr(V=3000, E=40000, seed=11):
    """A random directed graph (sorted, deduplicated rows) where ~1/4 of the vertices have no
    out-edges: regions of bias 0 (deg(u) = 0), rows whose every region is empty (T = 0: the walk
    ends, R20), and isolated seeds."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, V, E)
    dst = rng.integers(0, V, E)
    sink = rng.random(V) < 0.25
    keep = ~sink[src] & (src != dst)
    pairs = np.unique(np.stack([src[keep], dst[keep]], 1), axis=0)
    rp = np.zeros(V + 1, np.int64)
    np.add.at(rp, pairs[:, 0] + 1, 1)
    return np.cumsum(rp), pairs[:, 1].astype(np.uint32)


def test_buckets_directed_empty_regions():
    rp, col = directed_csr()
    Gb, Gh, og = graphs(rp, col)
    assert Gb.info()["walk_buckets"] == 1
    seeds = np.arange(0, len(rp) - 1, 3, dtype=np.uint32)
    pb = check_walk(Gb, og, "degree", seeds, 120, rng_seed=12)
    ph = u32(cs.csaw_walk(Gh, "degree", torch.as_tensor(seeds.view(np.int32)).to(DEV), 120, rng_seed=12))
    assert np.array_equal(pb, ph)
    assert (pb == cs.NONE).any(), "expected walks that end (rows without positive-bias neighbours)"
    Gb.close(); Gh.close()


def test_weight_buckets_directed_zero_rows():
    rp, col = directed_csr(seed=13)
    rng = np.random.default_rng(5)
    w = (rng.integers(1, 1 << 16, len(col)) * 2.0 ** -20).astype(np.float32)
    w[rng.random(len(col)) < 0.3] = 0.0          # zero weights, whole zero rows
    G, og = weighted(rp, col, w)
    assert G.info()["walk_buckets"] & 2
    seeds = np.arange(0, len(rp) - 1, 3, dtype=np.uint32)
    p = check_weight_exact(G, og, seeds, 120, 14, range(len(seeds)))
    assert (p == cs.NONE).any()
    G.close()


def test_buckets_short_and_empty_calls():
    g = rmat_csr(1 << 12, 1 << 16, 3, device=DEV).to("cpu")
    Gb, Gh, og = graphs(g.row_ptr, g.col_idx)
    seeds = instance_seeds(g, 40, set_id=5).numpy()
    for L in (0, 1, 31, 32, 33):
        check_walk(Gb, og, "degree", seeds, L, rng_seed=2)
    empty = torch.empty(0, dtype=torch.int32, device=DEV)
    assert cs.csaw_walk(Gb, "degree", empty, 10, rng_seed=1).shape == (0, 11)
    Gb.close(); Gh.close()


def test_weight_buckets_fall_back_outside_their_range():
    """Weights whose mean region width is below 2^-24 (here ~1e-30) cannot be bucketed (k out of
    [-24, 7]): the graph is created without the weighted index and walks take the per-step scan."""
    g = rmat_csr(1 << 12, 1 << 16, 3, device=DEV).to("cpu")
    w = torch.full((g.col_idx.numel(),), 1e-30, dtype=torch.float32)
    G, og = weighted(g.row_ptr, g.col_idx, w)
    assert not (G.info()["walk_buckets"] & 2)
    seeds = instance_seeds(g, 32, set_id=1).numpy()
    check_weight_exact(G, og, seeds, 20, 3, range(32))   # equal weights: every boundary is far from the draws
    G.close()
