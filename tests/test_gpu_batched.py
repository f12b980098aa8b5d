"""The two sampling drivers -- fused one-warp-per-instance (default for small
frontiers) and the level-synchronous batched queue -- must both match
the oracle and each other exactly (draws are keyed by (instance, depth, vertex))."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import instance_seeds, rmat_csr
from tests._golden import gtoy
from tests._parity import DEV, check_sample

pytestmark = pytest.mark.gpu


def batched_pair(row_ptr, col, cache=False):
    rp = torch.as_tensor(np.asarray(row_ptr, dtype=np.int64))
    c = torch.as_tensor(np.asarray(col).astype(np.uint32).view(np.int32))
    G = cs.csaw_graph_create(rp.to(DEV), c.to(DEV), batched_only=True, ctps_cache=cache)
    return G, O.Graph(rp.numpy(), c.numpy().view(np.uint32))


@pytest.fixture(scope="module")
def cfg1b():
    g = rmat_csr(1024, 16384, 1)
    G, og = batched_pair(g.row_ptr, g.col_idx)
    return G, og, g


@pytest.mark.parametrize("workload,fanout,a_max", [("degree", [2, 2], 0), ("uniform", [3, 2], 0),
                                                   ("degree", [8, 4], 2), ("layer", [2, 2], 0), ("layer", [4, 3], 2)])
def test_batched_driver_parity(cfg1b, workload, fanout, a_max):
    G, og, g = cfg1b
    check_sample(G, og, workload, instance_seeds(g, 300, set_id=4).numpy(), fanout=fanout, rng_seed=13, a_max=a_max)


def test_batched_driver_forest_fire(cfg1b):
    G, og, g = cfg1b
    check_sample(G, og, "forest_fire", instance_seeds(g, 300).numpy(), depth=3, pf=0.8, rng_seed=2)


def test_batched_gtoy():
    rp, col = gtoy()
    G, og = batched_pair(rp, col)
    seeds = np.tile(np.arange(12, dtype=np.uint32), 100)
    check_sample(G, og, "degree", seeds, fanout=[3, 2], rng_seed=5, a_max=2)
    check_sample(G, og, "layer", seeds, fanout=[3, 4], rng_seed=7)
    G.close()


@pytest.mark.parametrize("cache", [False, True])
def test_fused_equals_batched_medium(cache):
    g = rmat_csr(1 << 15, 1 << 19, 7, device=DEV)
    A = cs.csaw_graph_create(g.row_ptr, g.col_idx, ctps_cache=cache)
    B = cs.csaw_graph_create(g.row_ptr, g.col_idx, ctps_cache=cache, batched_only=True)
    seeds = instance_seeds(g, 4096).to(DEV)
    cases = [("degree", dict(fanout=[2, 2])), ("uniform", dict(fanout=[4, 3, 2])), ("layer", dict(fanout=[2, 2])),
             ("layer", dict(fanout=[8, 4, 2])), ("degree", dict(fanout=[10, 5]))]
    for kind, kw in cases:
        ra = cs.csaw_sample(A, kind, seeds, rng_seed=21, **kw)
        rb = cs.csaw_sample(B, kind, seeds, rng_seed=21, **kw)
        for x, y in zip(ra, rb):
            assert torch.equal(x, y), kind
    ff = cs.make_bias("forest_fire", pf=0.7)
    ra = cs.csaw_sample(A, ff, seeds, depth=2, rng_seed=3)
    rb = cs.csaw_sample(B, ff, seeds, depth=2, rng_seed=3)
    for x, y in zip(ra, rb):
        assert torch.equal(x, y)
    A.close()
    B.close()


@pytest.mark.parametrize("migration", ["repeated", "updated"])
@pytest.mark.parametrize("batched", [False, True])
def test_migration_baselines_parity(migration, batched):
    """NEXT-2 ablation modes (Fig. 6(a)/(b)) are bit-exact with the oracle too."""
    g = rmat_csr(1024, 16384, 1)
    rp = g.row_ptr.to(DEV)
    G = cs.csaw_graph_create(rp, g.col_idx.to(DEV), batched_only=batched)
    og = O.Graph.from_torch(g)
    seeds = instance_seeds(g, 300, set_id=6).numpy()
    check_sample(G, og, "degree", seeds, fanout=[8, 4], rng_seed=3, migration=migration)
    check_sample(G, og, "layer", seeds, fanout=[4, 3], rng_seed=3, migration=migration)
    check_sample(G, og, "uniform", seeds, fanout=[40, 3], rng_seed=3, migration=migration, a_max=4)
    G.close()
    rp_t, col_t = gtoy()
    G2 = cs.csaw_graph_create(torch.tensor(rp_t).to(DEV), torch.tensor(col_t.view(np.int32)).to(DEV),
                              batched_only=batched)
    check_sample(G2, O.Graph(rp_t, col_t), "degree", np.tile(np.arange(12, dtype=np.uint32), 50), fanout=[3, 2],
                 rng_seed=5, migration=migration, a_max=2)
    G2.close()
