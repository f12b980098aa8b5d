"""node2vec with per-edge triangle counts (capi.cu build_tri, walk.cu k_node2vec_tri):
T in closed form from |N(v) ∩ N(prev)| and a partial scan of N(v) from the end nearer
to the draw.  Must be bit-identical to the oracle's scanned CTPS (north star) for
balanced and very unequal list sizes, both scan directions, other integer (p, q)
scales, and must not be used on asymmetric graphs."""
import numpy as np
import pytest
import torch

import paper_2009_09103_b200 as cs
from synth import instance_seeds, rmat_csr
from tests._golden import gtoy
from tests._parity import DEV, check_walk, u32
from tests.test_gpu_parity import hub_csr

import oracle as O

pytestmark = pytest.mark.gpu


def cached(rp, col):
    rpt = torch.as_tensor(np.asarray(rp, dtype=np.int64))
    ct = torch.as_tensor(np.asarray(col).astype(np.uint32).view(np.int32))
    G = cs.csaw_graph_create(rpt.to(DEV), ct.to(DEV), node2vec_tri=True)
    return G, O.Graph(rpt.numpy(), ct.numpy().view(np.uint32))


@pytest.fixture(scope="module")
def medium():
    g = rmat_csr(1 << 15, 1 << 19, 7, device=DEV).to("cpu")
    G, og = cached(g.row_ptr, g.col_idx)
    assert G.info()["node2vec_tri"] == 1
    return G, og, g


@pytest.mark.parametrize("p,q", [(2.0, 0.5), (0.25, 4.0), (1.0, 1.0), (0.5, 2.0)])
def test_tri_medium(medium, p, q):
    G, og, g = medium
    seeds = instance_seeds(g, 192, set_id=4).numpy()
    check_walk(G, og, "node2vec", seeds, 60, rng_seed=13, p=p, q=q)
    st = cs.csaw_stats(G)
    assert st["index_bytes"] > 0


def test_tri_dense_rmat():
    # denser graph: long balanced lists (tile merges over several N(prev) windows)
    g = rmat_csr(1 << 12, 1 << 20, 11, device=DEV).to("cpu")
    G, og = cached(g.row_ptr, g.col_idx)
    seeds = instance_seeds(g, 96, set_id=1).numpy()
    check_walk(G, og, "node2vec", seeds, 40, rng_seed=3, p=2.0, q=0.5, instance_base=777)
    G.close()


def test_tri_hub():
    # d = 300,000 hub next to degree-3 ring vertices: per-key binary searches of N(prev)
    rp, col = hub_csr()
    G, og = cached(rp, col)
    seeds = np.array([0, 1, 0, 1, 5, 0, 1, 17, 299_999, 20_001], dtype=np.uint32)
    check_walk(G, og, "node2vec", seeds, 30, rng_seed=9, p=2.0, q=0.5)
    check_walk(G, og, "node2vec", seeds, 30, rng_seed=10, p=0.25, q=4.0)
    G.close()


def test_tri_gtoy_many_walkers():
    rp, col = gtoy()
    G, og = cached(rp, col)
    assert G.info()["node2vec_tri"] == 1
    seeds = np.tile(np.arange(12, dtype=np.uint32), 300)
    check_walk(G, og, "node2vec", seeds, 33, rng_seed=2, p=2.0, q=0.5)
    G.close()


def test_tri_not_built_for_asymmetric():
    rp = np.array([0, 2, 3, 4, 5], np.int64)      # 0 -> {1, 2}; 1 -> {0}; 2 -> {3}; 3 -> {0}
    col = np.array([1, 2, 0, 3, 0], np.uint32)
    G, og = cached(rp, col)
    assert G.info()["node2vec_tri"] == 0
    check_walk(G, og, "node2vec", np.array([0, 1, 2, 3], np.uint32), 9, rng_seed=1, p=2.0, q=0.5)
    G.close()


def test_tri_equals_uncached_large_batch():
    g = rmat_csr(1 << 16, 1 << 20, 5, device=DEV)
    seeds = instance_seeds(g, 20_000, set_id=2).to(DEV)
    G1 = cs.csaw_graph_create(g.row_ptr, g.col_idx, node2vec_tri=True)
    G2 = cs.csaw_graph_create(g.row_ptr, g.col_idx)
    b = cs.make_bias("node2vec", p=2.0, q=0.5)
    assert torch.equal(cs.csaw_walk(G1, b, seeds, 25, rng_seed=4), cs.csaw_walk(G2, b, seeds, 25, rng_seed=4))
    G1.close()
    G2.close()
