"""Out-of-memory mode (§5) for batched traversal sampling (neighbor sampling and
forest fire): each level's queue is grouped by owner partition and sampled
partition by partition.  Draws are keyed by (instance, depth, slot),
so the result must equal the in-memory run exactly and the oracle per instance."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import instance_seeds, rmat_csr
from tests._golden import gtoy
from tests._parity import DEV, check_sample

pytestmark = pytest.mark.gpu


def oom_budget(g, P, R):
    V = g.row_ptr.numel() - 1
    rp = g.row_ptr.cpu().numpy()
    bounds = O.partition_bounds(V, P)
    maxpe = max(int(rp[bounds[p + 1]] - rp[bounds[p]]) for p in range(P))
    return 8 * (V + 1) + 4 * V + R * maxpe * 4 + (1 << 20)


@pytest.fixture(scope="module")
def medium():
    return rmat_csr(1 << 15, 1 << 19, 7, device=DEV).to("cpu")


def _run(G, kind, seeds, fanout, depth, pf=0.0, migration="brs"):
    b = cs.make_bias(kind, pf=pf, migration=migration)
    return cs.csaw_sample(G, b, seeds, fanout=fanout, depth=depth, rng_seed=3, instance_base=5)


@pytest.mark.parametrize("P,R,S", [(4, 2, 2), (3, 1, 1), (7, 3, 2), (1, 1, 1)])
@pytest.mark.parametrize("kind", ["degree", "uniform", "forest_fire"])
def test_oom_sample_equals_in_memory(medium, P, R, S, kind):
    g = medium
    seeds = instance_seeds(g, 500, set_id=2).to(DEV)
    fan, depth, pf = ([], 3, 0.7) if kind == "forest_fire" else ([3, 2, 2], 3, 0.0)
    Gm = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV))
    ref = _run(Gm, kind, seeds, fan, depth, pf)
    Go = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=oom_budget(g, P, R), num_partitions=P,
                              max_resident=R, num_streams=S)
    assert Go.info()["oom_mode"] == 1
    got = _run(Go, kind, seeds, fan, depth, pf)
    torch.cuda.synchronize()
    for a, b in zip(ref, got):
        assert torch.equal(a.cpu(), b.cpu())
    st = cs.csaw_stats(Go)
    assert st["sampled_edges"] == got[1].numel()
    assert st["partition_loads"] >= 1
    if P > R:
        assert st["partition_loads"] > R          # partitions were swapped between waves
    # repeated call: residents persist and the result is unchanged
    again = _run(Go, kind, seeds, fan, depth, pf)
    for a, b in zip(ref, again):
        assert torch.equal(a.cpu(), b.cpu())
    Gm.close()
    Go.close()


def test_oom_sample_oracle_and_migration(medium):
    g = medium
    og = O.Graph(g.row_ptr.numpy(), g.col_idx.numpy().view(np.uint32))
    seeds = instance_seeds(g, 120, set_id=4).numpy()
    Go = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=oom_budget(g, 5, 2), num_partitions=5,
                              max_resident=2)
    for mig in ("brs", "repeated", "updated"):
        _, total = check_sample(Go, og, "degree", seeds, fanout=(8, 4), rng_seed=9, migration=mig)
        assert total > 0
    Go.close()


def test_oom_sample_gtoy_fig8():
    """G_toy in 3 partitions with 2 resident (Fig. 8), every seed, vs the oracle."""
    rp, col = gtoy()
    og = O.Graph(rp, col)
    V = len(rp) - 1
    Go = cs.csaw_graph_create(torch.tensor(rp), torch.tensor(col.view(np.int32)), budget_bytes=1 << 20,
                              num_partitions=3, max_resident=2)
    assert Go.info()["oom_mode"] == 1
    seeds = np.array([v for v in range(V) if rp[v + 1] > rp[v]] * 3, dtype=np.uint32)
    check_sample(Go, og, "degree", seeds, fanout=(2, 2, 2), rng_seed=4)
    check_sample(Go, og, "forest_fire", seeds, depth=3, pf=0.6, rng_seed=4)
    Go.close()


def test_oom_sample_unsupported(medium):
    g = medium
    Go = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=oom_budget(g, 4, 2), num_partitions=4,
                              max_resident=2)
    s = instance_seeds(g, 4).to(DEV)
    with pytest.raises(cs.CsawError):
        cs.csaw_sample(Go, cs.make_bias("layer"), s, fanout=[2])
    Go.close()


@pytest.mark.parametrize("kind", ["degree", "forest_fire", "layer"])
def test_oom_zerocopy_sample_equals_in_memory(medium, kind):
    """NEXT-4(ii) for traversal sampling: col_idx read in place from pinned host memory."""
    g = medium
    seeds = instance_seeds(g, 400, set_id=6).to(DEV)
    fan, depth, pf = {"degree": ([4, 3], 2, 0.0), "forest_fire": ([], 3, 0.7), "layer": ([3, 3], 2, 0.0)}[kind]
    Gm = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV))
    ref = _run(Gm, kind, seeds, fan, depth, pf)
    Gz = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=oom_budget(g, 4, 1), num_partitions=4,
                              max_resident=1, zerocopy=True)
    got = _run(Gz, kind, seeds, fan, depth, pf)
    for a, b in zip(ref, got):
        assert torch.equal(a.cpu(), b.cpu())
    assert cs.csaw_stats(Gz)["partition_loads"] == 0
    Gm.close()
    Gz.close()


def test_oom_snowball_equals_in_memory(medium):
    g = medium
    seeds = instance_seeds(g, 40, set_id=8).to(DEV)
    Gm = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV))
    ref = _run(Gm, "snowball", seeds, [], 2)
    Go = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=oom_budget(g, 4, 2), num_partitions=4,
                              max_resident=2)
    got = _run(Go, "snowball", seeds, [], 2)
    for a, b in zip(ref, got):
        assert torch.equal(a.cpu(), b.cpu())
    Gm.close()
    Go.close()
