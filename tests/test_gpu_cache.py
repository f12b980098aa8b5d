"""Static-bias CTPS cache (CSAW_GRAPH_CTPS_CACHE, §8(f) NEXT-1; the paper's deleted
"caching transition probability"): every degree-biased selection must
be bit-identical to the oracle (and therefore to the scanned path)."""
import numpy as np
import pytest
import torch

import paper_2009_09103_b200 as cs
from synth import CONFIGS, instance_seeds, rmat_csr
from tests._golden import gtoy
from tests._parity import DEV, check_sample, check_walk, u32
from tests.test_gpu_parity import hub_csr

import oracle as O

pytestmark = pytest.mark.gpu


def cached_pair(row_ptr, col):
    rp = torch.as_tensor(np.asarray(row_ptr, dtype=np.int64))
    c = torch.as_tensor(np.asarray(col).astype(np.uint32).view(np.int32))
    G = cs.csaw_graph_create(rp.to(DEV), c.to(DEV), ctps_cache=True)
    assert G.info()["ctps_cache"] == 1
    return G, O.Graph(rp.numpy(), c.numpy().view(np.uint32))


@pytest.fixture(scope="module")
def cfg1c():
    g = rmat_csr(1024, 16384, 1)
    G, og = cached_pair(g.row_ptr, g.col_idx)
    return G, og, g


@pytest.fixture(scope="module")
def hubc():
    return cached_pair(*hub_csr())


@pytest.mark.parametrize("rng_seed", [1, 2, 3])
def test_cfg1_cached(cfg1c, rng_seed):
    G, og, g = cfg1c
    check_sample(G, og, "degree", instance_seeds(g, 64).numpy(), fanout=[2, 2], rng_seed=rng_seed)
    st = cs.csaw_stats(G)
    assert st["cache_probes"] > 0 and st["neighbours_scanned"] == 0


@pytest.mark.parametrize("workload,fanout,a_max", [("degree", [5, 3, 2], 0), ("degree", [40], 0),
                                                   ("degree", [8, 4], 2), ("degree", [70, 40], 2),
                                                   ("layer", [2, 2], 0), ("layer", [4, 3], 2), ("layer", [40, 2], 0)])
def test_cached_variants(cfg1c, workload, fanout, a_max):
    G, og, g = cfg1c
    check_sample(G, og, workload, instance_seeds(g, 300, set_id=5).numpy(), fanout=fanout, rng_seed=11, a_max=a_max)


def test_cached_gtoy_collisions():
    rp, col = gtoy()
    G, og = cached_pair(rp, col)
    seeds = np.tile(np.arange(12, dtype=np.uint32), 200)
    for a_max in (0, 2):
        check_sample(G, og, "degree", seeds, fanout=[3, 2], rng_seed=5, a_max=a_max)
        check_sample(G, og, "layer", seeds, fanout=[3, 4], rng_seed=7, a_max=a_max)
    G.close()


def test_cached_walks(cfg1c):
    G, og, g = cfg1c
    check_walk(G, og, "degree", instance_seeds(g, 64).numpy(), 300, rng_seed=4)
    check_walk(G, og, "uniform", instance_seeds(g, 64).numpy(), 100, rng_seed=4)


def test_cached_hub_pools(hubc):
    G, og = hubc
    seeds = np.array([0, 1, 0, 1, 5, 0, 1, 17], dtype=np.uint32)
    check_sample(G, og, "degree", seeds, fanout=[40, 2], rng_seed=3)
    check_sample(G, og, "degree", seeds, fanout=[3, 2], rng_seed=4, a_max=2)
    check_sample(G, og, "layer", seeds, fanout=[2, 2], rng_seed=7)
    check_walk(G, og, "degree", seeds, 20, rng_seed=8)


def test_cached_equals_scanned_medium():
    g = rmat_csr(1 << 15, 1 << 19, 7, device=DEV)
    A = cs.csaw_graph_create(g.row_ptr, g.col_idx)
    B = cs.csaw_graph_create(g.row_ptr, g.col_idx, ctps_cache=True)
    seeds = instance_seeds(g, 2048).to(DEV)
    assert torch.equal(cs.csaw_walk(A, "degree", seeds, 200, rng_seed=9), cs.csaw_walk(B, "degree", seeds, 200, rng_seed=9))
    for kind, fan in (("degree", [2, 2]), ("layer", [2, 2])):
        ra = cs.csaw_sample(A, kind, seeds, fanout=fan, rng_seed=9)
        rb = cs.csaw_sample(B, kind, seeds, fanout=fan, rng_seed=9)
        for x, y in zip(ra, rb):
            assert torch.equal(x, y)
    A.close()
    B.close()


@pytest.mark.slow
def test_cfg2_cached_full():
    cfg = CONFIGS["cfg2"]
    g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=DEV)
    G = cs.csaw_graph_create(g.row_ptr, g.col_idx, ctps_cache=True)
    og = O.Graph(g.row_ptr.cpu().numpy(), g.col_idx.cpu().numpy().view(np.uint32))
    seeds = instance_seeds(g, cfg.n_instances).to(DEV)
    path = u32(cs.csaw_walk(G, "degree", seeds, cfg.length, rng_seed=1))
    sv = u32(seeds)
    for w in (0, 1, 1000, 2047, 3999):
        assert np.array_equal(path[w], O.walk(og, O.KIND_DEGREE, cfg.length, int(sv[w]), w, 1)), w
    G.close()


@pytest.mark.parametrize("heads", [True, False])
def test_cached_sampling_heads_vs_btree(hubc, heads):
    """Cached degree / layer pools search the vertex heads (wix.cuh) when the walk index
    exists; CSAW_GRAPH_SAMPLE_NO_HEADS forces the u64 B-tree.  Both bit-exact."""
    G, og = hubc
    assert G.info()["walk_index_heads"] == 1
    if not heads:
        G = cs.csaw_graph_create(torch.as_tensor(og.row_ptr).to(DEV),
                                 torch.as_tensor(og.col.view(np.int32)).to(DEV), ctps_cache=True,
                                 flags=cs.CSAW_GRAPH_SAMPLE_NO_HEADS)
    seeds = np.array([0, 1, 0, 1, 5, 0, 1, 17, 299_999, 20_000], dtype=np.uint32)
    check_sample(G, og, "degree", seeds, fanout=[30, 3], rng_seed=41)
    check_sample(G, og, "degree", seeds, fanout=[3, 2], rng_seed=42, a_max=2)
    check_sample(G, og, "layer", seeds, fanout=[3, 4], rng_seed=43)
