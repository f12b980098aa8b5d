"""Out-of-memory mode (§5): partitioned MDRW under an imposed device budget must
equal the in-memory run exactly (draws are keyed by (instance, step), R7/R22),
and the oracle on sampled instances."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import mdrw_seeds, rmat_csr
from tests._golden import gtoy
from tests._parity import DEV, u32

pytestmark = pytest.mark.gpu


def budget_for(g, P, R, n, m):
    V = g.row_ptr.numel() - 1
    rp = g.row_ptr.cpu().numpy()
    bounds = O.partition_bounds(V, P)
    maxpe = max(int(rp[bounds[p + 1]] - rp[bounds[p]]) for p in range(P))
    nblk = (m + 31) // 32
    state = n * m * 8 + n * nblk * 8 + n * 16 + 2 * P * n * 4 + 2 * P * 4 + 64 + 1024
    return 8 * (V + 1) + 4 * V + R * maxpe * 4 + state


@pytest.fixture(scope="module")
def medium():
    return rmat_csr(1 << 15, 1 << 19, 7, device=DEV).to("cpu")


@pytest.mark.parametrize("P,R,S", [(4, 2, 2), (3, 1, 1), (5, 3, 2), (1, 1, 1)])
def test_oom_mdrw_equals_in_memory(medium, P, R, S):
    g = medium
    n, m, L = 64, 200, 300
    seeds = mdrw_seeds(g, n, m).to(DEV)
    Gm = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV))
    ref = cs.csaw_walk(Gm, cs.make_bias("mdrw"), seeds, L, rng_seed=5)
    Go = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=budget_for(g, P, R, n, m), num_partitions=P,
                              max_resident=R, num_streams=S)
    assert Go.info()["oom_mode"] == 1
    got = cs.csaw_walk(Go, cs.make_bias("mdrw"), seeds, L, rng_seed=5)
    torch.cuda.synchronize()
    assert torch.equal(ref, got)
    st = cs.csaw_stats(Go)
    assert st["partition_loads"] >= min(P, 1) and st["sampled_edges"] == n * L
    if P > R:
        assert st["partition_loads"] > R            # partitions were swapped
    og = O.Graph(g.row_ptr.numpy(), g.col_idx.numpy().view(np.uint32))
    e = u32(got)
    sv = u32(seeds)
    for i in (0, 17, 63):
        assert np.array_equal(e[i], O.mdrw(og, sv[i], L, i, 5))
    Gm.close()
    Go.close()


def test_oom_gtoy_fig8_partitions():
    """Fig. 8 setup: G_toy in 3 partitions, 2 resident."""
    rp, col = gtoy()
    rpt = torch.tensor(rp)
    colt = torch.tensor(col.view(np.int32))
    seeds = torch.tensor([[0, 2, 8], [8, 0, 3], [4, 4, 11]], dtype=torch.int32, device=DEV)
    Gm = cs.csaw_graph_create(rpt.to(DEV), colt.to(DEV))
    Go = cs.csaw_graph_create(rpt, colt, budget_bytes=1 << 20, num_partitions=3, max_resident=2, num_streams=2)
    a = cs.csaw_walk(Gm, cs.make_bias("mdrw"), seeds, 40, rng_seed=2)
    b = cs.csaw_walk(Go, cs.make_bias("mdrw"), seeds, 40, rng_seed=2)
    assert torch.equal(a, b)
    Gm.close()
    Go.close()


def test_oom_budget_enforced(medium):
    g = medium
    with pytest.raises(cs.CsawError) as ei:
        cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=1 << 16, num_partitions=4, max_resident=2)
    assert ei.value.status == 6
    # graph fits but instance state does not
    Go = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=budget_for(g, 4, 2, 1, 1), num_partitions=4,
                              max_resident=2)
    seeds = mdrw_seeds(g, 256, 500).to(DEV)
    with pytest.raises(cs.CsawError) as ei:
        cs.csaw_walk(Go, cs.make_bias("mdrw"), seeds, 10)
    assert ei.value.status == 6
    Go.close()


def test_oom_zerocopy_equals_in_memory(medium):
    """NEXT-4(ii): col_idx read in place from pinned host memory under the budget."""
    g = medium
    n, m, L = 64, 200, 300
    seeds = mdrw_seeds(g, n, m).to(DEV)
    Gm = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV))
    Gz = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=budget_for(g, 4, 1, n, m), num_partitions=4,
                              max_resident=1, zerocopy=True)
    assert torch.equal(cs.csaw_walk(Gm, cs.make_bias("mdrw"), seeds, L, rng_seed=5),
                       cs.csaw_walk(Gz, cs.make_bias("mdrw"), seeds, L, rng_seed=5))
    s1 = seeds[:, 0].contiguous()
    assert torch.equal(cs.csaw_walk(Gm, "uniform", s1, L, rng_seed=6), cs.csaw_walk(Gz, "uniform", s1, L, rng_seed=6))
    assert torch.equal(cs.csaw_walk(Gm, "degree", s1, 60, rng_seed=7), cs.csaw_walk(Gz, "degree", s1, 60, rng_seed=7))
    Gm.close()
    Gz.close()


@pytest.mark.parametrize("kind", ["degree", "uniform"])
@pytest.mark.parametrize("P,R,S,ws,bal", [(4, 2, 2, True, True), (3, 1, 1, True, True), (5, 2, 2, False, True),
                                          (4, 2, 2, True, False), (4, 2, 1, False, False)])
def test_oom_walk_equals_in_memory(medium, kind, P, R, S, ws, bal):
    """Fig. 13(b) workload: degree-biased / uniform walks under partition scheduling
    (walkers migrate between per-partition queues); schedule switches never change results."""
    g = medium
    seeds = mdrw_seeds(g, 300, 1)[:, 0].contiguous().to(DEV)
    L = 120
    Gm = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV))
    ref = cs.csaw_walk(Gm, kind, seeds, L, rng_seed=4, instance_base=9)
    Go = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=budget_for(g, P, R, 1, 1) + (1 << 20),
                              num_partitions=P, max_resident=R, num_streams=S, oom_ws=ws, oom_bal=bal)
    got = cs.csaw_walk(Go, kind, seeds, L, rng_seed=4, instance_base=9)
    assert torch.equal(ref, got)
    st = cs.csaw_stats(Go)
    assert st["sampled_edges"] == 300 * L and st["partition_loads"] >= 1
    if kind == "degree":
        assert st["neighbours_scanned"] > 0
    Gm.close()
    Go.close()


@pytest.mark.parametrize("ws,bal", [(False, True), (True, False), (False, False)])
def test_oom_schedule_switches_keep_results(medium, ws, bal):
    g = medium
    n, m, L = 32, 100, 150
    seeds = mdrw_seeds(g, n, m).to(DEV)
    Gm = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV))
    Go = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=budget_for(g, 4, 2, n, m), num_partitions=4,
                              max_resident=2, oom_ws=ws, oom_bal=bal)
    assert torch.equal(cs.csaw_walk(Gm, cs.make_bias("mdrw"), seeds, L, rng_seed=5),
                       cs.csaw_walk(Go, cs.make_bias("mdrw"), seeds, L, rng_seed=5))
    s1 = seeds[:, 0].contiguous()
    a = cs.csaw_sample(Gm, "degree", s1, fanout=[4, 3], rng_seed=2)
    b = cs.csaw_sample(Go, "degree", s1, fanout=[4, 3], rng_seed=2)
    for x, y in zip(a, b):
        assert torch.equal(x.cpu(), y.cpu())
    Gm.close()
    Go.close()


@pytest.mark.parametrize("frac", [0.0, 0.3, 0.7, 1.2])   # 0.0: the smallest budget that validates
def test_oom_zerocopy_resident_prefix(medium, frac):
    """Zero-copy mode keeps col_idx[0, colc) on the device, colc = (budget - row_ptr - deg -
    min(512 MiB, budget/8)) / 4: MDRW steps read entries below colc from HBM and the rest
    from pinned host memory.  Budgets giving 0 %, ~30 %, ~70 % and 100 % resident must all
    equal the in-memory result (and the oracle)."""
    import os
    g = medium
    n, m, L = 48, 150, 250
    V, E = g.row_ptr.numel() - 1, g.col_idx.numel()
    resident = 8 * (V + 1) + 4 * V
    budget = max(int((resident + frac * 4 * E) * 8 / 7) + 64, budget_for(g, 4, 1, n, m))   # >= validation slot
    seeds = mdrw_seeds(g, n, m).to(DEV)
    Gm = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV))
    Gz = cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=budget, num_partitions=4, max_resident=1,
                              zerocopy=True)
    held = Gz.info()["device_bytes"]
    assert held <= budget
    if 0 < frac < 1:   # a partial resident prefix: both the HBM and the host branch are taken
        assert resident + 4 * E * frac * 0.5 < held < resident + 4 * E
    ref = cs.csaw_walk(Gm, cs.make_bias("mdrw"), seeds, L, rng_seed=9)
    assert torch.equal(ref, cs.csaw_walk(Gz, cs.make_bias("mdrw"), seeds, L, rng_seed=9))
    og = O.Graph(g.row_ptr.numpy(), g.col_idx.numpy().view(np.uint32))
    e = u32(ref)
    sv = u32(seeds.cpu())
    for i in (0, n // 2, n - 1):
        assert np.array_equal(e[i], O.mdrw(og, sv[i], L, i, 9))
    Gm.close()
    Gz.close()
