"""node2vec with the per-edge intersection index (n2v_index.cu, CSAW_GRAPH_N2V_INDEX):
a binary search over the positions of N(v) ∩ N(prev) in N(v) and a closed form between
them.  Must be bit-identical to the oracle's scanned CTPS (north star) on both sides of
prev, for members-free edges, hubs, other integer (p, q) scales, and must not be used on
asymmetric graphs."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import instance_seeds, rmat_csr
from tests._golden import gtoy
from tests._parity import DEV, check_walk
from tests.test_gpu_parity import hub_csr

pytestmark = pytest.mark.gpu


def indexed(rp, col):
    rpt = torch.as_tensor(np.asarray(rp, dtype=np.int64))
    ct = torch.as_tensor(np.asarray(col).astype(np.uint32).view(np.int32))
    G = cs.csaw_graph_create(rpt.to(DEV), ct.to(DEV), node2vec_index=True)
    return G, O.Graph(rpt.numpy(), ct.numpy().view(np.uint32))


@pytest.fixture(scope="module")
def medium():
    g = rmat_csr(1 << 15, 1 << 19, 7, device=DEV).to("cpu")
    G, og = indexed(g.row_ptr, g.col_idx)
    assert G.info()["node2vec_index"] == 1
    return G, og, g


# integer scales (R16): (wp, w1, wq) = (1, 2, 4), (16, 4, 1), (1, 1, 1), (4, 2, 1), (1, 4, 4) and, with a wq
# that is not a power of two (the quotient by fp64 estimate + correction, not a shift), (1, 3, 3), (1, 5, 10)
@pytest.mark.parametrize("p,q", [(2.0, 0.5), (0.25, 4.0), (1.0, 1.0), (0.5, 2.0), (4.0, 1.0), (3.0, 1.0), (5.0, 0.5)])
def test_index_medium(medium, p, q):
    G, og, g = medium
    seeds = instance_seeds(g, 256, set_id=4).numpy()
    check_walk(G, og, "node2vec", seeds, 60, rng_seed=13, p=p, q=q)
    st = cs.csaw_stats(G)
    assert st["pools"] > 0 and st["index_bytes"] > 0


def test_index_dense_rmat():
    # dense graph: many common neighbours per edge (long member lists, deep searches)
    g = rmat_csr(1 << 12, 1 << 20, 11, device=DEV).to("cpu")
    G, og = indexed(g.row_ptr, g.col_idx)
    assert G.info()["node2vec_index"] == 1
    seeds = instance_seeds(g, 128, set_id=1).numpy()
    check_walk(G, og, "node2vec", seeds, 40, rng_seed=3, p=2.0, q=0.5, instance_base=777)
    G.close()


def test_index_hub():
    rp, col = hub_csr()
    G, og = indexed(rp, col)
    seeds = np.array([0, 1, 0, 1, 5, 0, 1, 17, 299_999, 20_001], dtype=np.uint32)
    check_walk(G, og, "node2vec", seeds, 30, rng_seed=9, p=2.0, q=0.5)
    check_walk(G, og, "node2vec", seeds, 30, rng_seed=10, p=0.25, q=4.0)
    check_walk(G, og, "node2vec", seeds, 30, rng_seed=11, p=5.0, q=0.5)
    G.close()


def test_index_gtoy_many_walkers():
    rp, col = gtoy()
    G, og = indexed(rp, col)
    assert G.info()["node2vec_index"] == 1
    seeds = np.tile(np.arange(12, dtype=np.uint32), 300)
    check_walk(G, og, "node2vec", seeds, 33, rng_seed=2, p=2.0, q=0.5)
    G.close()


def test_index_not_built_for_asymmetric():
    rp = np.array([0, 2, 3, 4, 5], np.int64)      # 0 -> {1, 2}; 1 -> {0}; 2 -> {3}; 3 -> {0}
    col = np.array([1, 2, 0, 3, 0], np.uint32)
    G, og = indexed(rp, col)
    assert G.info()["node2vec_index"] == 0
    check_walk(G, og, "node2vec", np.array([0, 1, 2, 3], np.uint32), 9, rng_seed=1, p=2.0, q=0.5)
    G.close()


def test_index_equals_tri_and_merge_large_batch():
    g = rmat_csr(1 << 16, 1 << 20, 5, device=DEV)
    seeds = instance_seeds(g, 50_000, set_id=2).to(DEV)
    Gx = cs.csaw_graph_create(g.row_ptr, g.col_idx, node2vec_index=True)
    Gt = cs.csaw_graph_create(g.row_ptr, g.col_idx, node2vec_tri=True)
    Gm = cs.csaw_graph_create(g.row_ptr, g.col_idx)
    for p, q in ((2.0, 0.5), (0.5, 2.0)):
        b = cs.make_bias("node2vec", p=p, q=q)
        x = cs.csaw_walk(Gx, b, seeds, 25, rng_seed=4, instance_base=1000)
        assert torch.equal(x, cs.csaw_walk(Gt, b, seeds, 25, rng_seed=4, instance_base=1000))
        assert torch.equal(x, cs.csaw_walk(Gm, b, seeds, 25, rng_seed=4, instance_base=1000))
    # float (p, q): the index is not used (integer path only); result equals the merge kernel
    b = cs.make_bias("node2vec", p=3.14159, q=2.71828)
    assert torch.equal(cs.csaw_walk(Gx, b, seeds[:500], 10, rng_seed=1), cs.csaw_walk(Gm, b, seeds[:500], 10, rng_seed=1))
    for G in (Gx, Gt, Gm):
        G.close()


def test_index_pinned_host_path_pipelined(medium):
    """A pinned host path: the walk runs in 8 walker ranges whose rows are copied back while the
    next range walks (g->copy_st); same rows as a device output and as the oracle."""
    G, og, g = medium
    seeds = instance_seeds(g, 4096, set_id=6).numpy()
    st = torch.as_tensor(seeds.view(np.int32)).to(DEV)
    dev = cs.csaw_walk(G, cs.make_bias("node2vec", p=2.0, q=0.5), st, 40, rng_seed=21)
    host = torch.empty_like(dev, device="cpu").pin_memory()
    cs.csaw_walk(G, cs.make_bias("node2vec", p=2.0, q=0.5), st.cpu().pin_memory(), 40, rng_seed=21, out=host)
    assert torch.equal(host, dev.cpu())
    check_walk(G, og, "node2vec", seeds, 40, rng_seed=21, p=2.0, q=0.5, walkers=range(0, 4096, 97))
    # a second call on another stream right after (shared scratch, copy stream ordering)
    s2 = torch.cuda.Stream(device=DEV)
    host2 = torch.empty_like(host).pin_memory()
    cs.csaw_walk(G, cs.make_bias("node2vec", p=2.0, q=0.5), st, 40, rng_seed=21, out=host2, stream=s2)
    s2.synchronize()
    assert torch.equal(host2, host)
