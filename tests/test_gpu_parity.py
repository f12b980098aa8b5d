"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Integer biases must match bit for bit (north star).  Sizes here let the oracle
finish in seconds while spanning many warps, multi-chunk CTPS tables, the
bitmap and list collision paths, multi-pass (k > 32) selection, the attempt-cap
fallback and ragged tails; full-size configs are in test_gpu_configs.py.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import instance_seeds, mdrw_seeds, rmat_csr
from tests._golden import gtoy, philox_kats
from tests._parity import DEV, check_mdrw, check_node2vec_float, check_sample, check_walk, graph_pair, u32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg1():
    g = rmat_csr(1024, 16384, 1)
    G, og = graph_pair(g.row_ptr, g.col_idx)
    return G, og, g


@pytest.fixture(scope="module")
def medium():
    g = rmat_csr(1 << 15, 1 << 19, 7, device=DEV).to("cpu")
    G, og = graph_pair(g.row_ptr, g.col_idx)
    return G, og, g


@pytest.fixture(scope="module")
def toy():
    rp, col = gtoy()
    return graph_pair(rp, col)


def hub_csr():
    """Vertex 0 adjacent to 1..300000 (d = 300000, chunked CTPS with m > U), vertex 1 to
    2..20001 (d = 20001 > bitmap bits: list path), plus a ring so every vertex has degree >= 2."""
    V = 300_001
    edges = set()
    for u in range(1, V):
        edges.add((0, u))
    for u in range(2, 20_002):
        edges.add((1, u))
    for u in range(1, V):
        w = u + 1 if u + 1 < V else 1
        edges.add((min(u, w), max(u, w)))
    e = np.array(sorted(edges), dtype=np.int64)
    src = np.concatenate([e[:, 0], e[:, 1]])
    dst = np.concatenate([e[:, 1], e[:, 0]])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    rp = np.zeros(V + 1, np.int64)
    np.add.at(rp, src + 1, 1)
    rp = np.cumsum(rp)
    return rp, dst.astype(np.uint32)


@pytest.fixture(scope="module")
def hub():
    rp, col = hub_csr()
    return graph_pair(rp, col)


# ------------------------------------------------------------------ RNG
@pytest.mark.parametrize("ctr,key,out", philox_kats())
def test_device_philox_kat(ctr, key, out):
    c = torch.tensor(np.array([ctr], dtype=np.uint32).view(np.int32))
    k = torch.tensor(np.array(key, dtype=np.uint32).view(np.int32))
    o = u32(cs.csaw_philox(c.to(DEV), k.to(DEV)))
    assert o[0].tolist() == out


def test_device_philox_matches_curand():
    assert cs.csaw_selftest_curand(1 << 22) == 0


def test_device_philox_matches_oracle_random_counters():
    rng = np.random.default_rng(3)
    c = rng.integers(0, 2**32, size=(4096, 4), dtype=np.uint64).astype(np.uint32)
    k = np.array([0xDEADBEEF, 0x12345678], np.uint32)
    o = u32(cs.csaw_philox(torch.tensor(c.view(np.int32)).to(DEV), torch.tensor(k.view(np.int32)).to(DEV)))
    for i in range(0, 4096, 97):
        assert o[i].tolist() == O.philox4x32_10(c[i].tolist(), k.tolist())


# ------------------------------------------------------------------ config 1 (full)
@pytest.mark.parametrize("rng_seed", [1, 2, 3])
def test_cfg1_degree_neighbor_sampling_full(cfg1, rng_seed):
    G, og, g = cfg1
    seeds = instance_seeds(g, 64).numpy()
    _, total = check_sample(G, og, "degree", seeds, fanout=[2, 2], rng_seed=rng_seed)
    assert total > 64


@pytest.mark.parametrize("workload,fanout,a_max", [
    ("uniform", [2, 2], 0), ("degree", [5, 3, 2], 0), ("degree", [40], 0), ("degree", [8, 4], 2),
    ("uniform", [33, 2], 0), ("degree", [0, 3], 0), ("degree", [70, 40], 2),
])
def test_neighbor_sampling_variants(cfg1, workload, fanout, a_max):
    G, og, g = cfg1
    seeds = instance_seeds(g, 300, set_id=5).numpy()
    check_sample(G, og, workload, seeds, fanout=fanout, rng_seed=11, a_max=a_max)


def test_gtoy_collision_heavy(toy):
    G, og = toy
    seeds = np.tile(np.arange(12, dtype=np.uint32), 200)
    for a_max in (0, 2):
        check_sample(G, og, "degree", seeds, fanout=[3, 2], rng_seed=5, a_max=a_max)
        check_sample(G, og, "uniform", seeds, fanout=[4, 2, 1], rng_seed=6, a_max=a_max)
        check_sample(G, og, "layer", seeds, fanout=[3, 4], rng_seed=7, a_max=a_max)


@pytest.mark.parametrize("pf,depth", [(0.7, 2), (0.95, 3), (0.0, 2)])
def test_forest_fire(cfg1, pf, depth):
    G, og, g = cfg1
    seeds = instance_seeds(g, 400, set_id=2).numpy()
    check_sample(G, og, "forest_fire", seeds, depth=depth, pf=pf, rng_seed=21)


@pytest.mark.parametrize("fanout", [[2, 2], [4, 3], [1, 1, 1], [40, 2]])
def test_layer_sampling(cfg1, fanout):
    G, og, g = cfg1
    seeds = instance_seeds(g, 256, set_id=3).numpy()
    check_sample(G, og, "layer", seeds, fanout=fanout, rng_seed=31)


def test_medium_graph_sampling(medium):
    G, og, g = medium
    seeds = instance_seeds(g, 512).numpy()
    check_sample(G, og, "degree", seeds, fanout=[2, 2], rng_seed=1)
    check_sample(G, og, "layer", seeds[:128], fanout=[2, 2], rng_seed=1)
    check_sample(G, og, "forest_fire", seeds, depth=2, pf=0.7, rng_seed=1)


def test_hub_pools(hub):
    """Pools of 300,000 / 20,001 candidates: chunked CTPS with rescans, list-based
    collision detection, k > 32 multi-pass selection and the attempt-cap fallback."""
    G, og = hub
    seeds = np.array([0, 1, 0, 1, 5, 0, 1, 17], dtype=np.uint32)
    check_sample(G, og, "degree", seeds, fanout=[40, 2], rng_seed=3)
    check_sample(G, og, "degree", seeds, fanout=[3, 2], rng_seed=4, a_max=2)
    check_sample(G, og, "uniform", seeds, fanout=[50, 1], rng_seed=5)
    check_sample(G, og, "forest_fire", seeds, depth=2, pf=0.9, rng_seed=6)
    check_sample(G, og, "layer", seeds, fanout=[2, 2], rng_seed=7)
    check_walk(G, og, "degree", seeds, 20, rng_seed=8)
    check_walk(G, og, "node2vec", seeds, 12, rng_seed=9, p=2.0, q=0.5)


# ------------------------------------------------------------------ walks
@pytest.mark.parametrize("kind", ["degree", "uniform"])
def test_walks_cfg1(cfg1, kind):
    G, og, g = cfg1
    seeds = instance_seeds(g, 64).numpy()
    check_walk(G, og, kind, seeds, 200, rng_seed=4)


@pytest.mark.parametrize("kind", ["degree", "uniform"])
def test_walks_medium(medium, kind):
    G, og, g = medium
    seeds = instance_seeds(g, 256).numpy()
    check_walk(G, og, kind, seeds, 300, rng_seed=2)


def test_node2vec_integer(medium):
    G, og, g = medium
    seeds = instance_seeds(g, 128).numpy()
    check_walk(G, og, "node2vec", seeds, 40, rng_seed=3, p=2.0, q=0.5)
    check_walk(G, og, "node2vec", seeds[:32], 20, rng_seed=3, p=0.25, q=4.0)


def test_node2vec_float_boundary_rule(medium):
    G, og, g = medium
    seeds = instance_seeds(g, 64).numpy()
    excused = check_node2vec_float(G, og, seeds, 30, math.pi, math.e, rng_seed=5)
    assert excused <= 2


def test_node2vec_p1q1_equals_uniform_walk(medium):
    G, og, g = medium
    seeds = torch.as_tensor(instance_seeds(g, 64).numpy()).to(DEV)
    a = cs.csaw_walk(G, cs.make_bias("node2vec", p=1.0, q=1.0), seeds, 50, rng_seed=9)
    b = cs.csaw_walk(G, "uniform", seeds, 50, rng_seed=9)
    assert torch.equal(a, b)


def test_mdrw(cfg1, medium):
    G, og, g = cfg1
    s = mdrw_seeds(g, 24, 50).numpy()
    check_mdrw(G, og, s, 300, rng_seed=2)
    G2, og2, g2 = medium
    s2 = mdrw_seeds(g2, 6, 2000).numpy()
    check_mdrw(G2, og2, s2, 500, rng_seed=3)
    s1 = mdrw_seeds(g2, 16, 1).numpy()
    e = check_mdrw(G2, og2, s1, 100, rng_seed=4)
    p = u32(cs.csaw_walk(G2, "uniform", torch.as_tensor(s1[:, 0].view(np.int32)).to(DEV), 100, rng_seed=4))
    assert np.array_equal(e[:, :, 0], p[:, :-1]) and np.array_equal(e[:, :, 1], p[:, 1:])


# ------------------------------------------------------------------ edge cases / boundary behaviour
def test_empty_and_degenerate(cfg1):
    G, og, g = cfg1
    empty = torch.empty(0, dtype=torch.int32, device=DEV)
    offs, src, dst, dep = cs.csaw_sample(G, "degree", empty, fanout=[2, 2])
    assert offs.numel() == 1 and int(offs[0]) == 0 and src.numel() == 0
    assert cs.csaw_walk(G, "degree", empty, 10).shape == (0, 11)
    # isolated seed: no edges; walk pads with NONE after the seed
    iso = int(torch.nonzero(g.degrees() == 0)[0])
    seeds = torch.tensor([iso, iso], dtype=torch.int32, device=DEV)
    offs, src, *_ = cs.csaw_sample(G, "degree", seeds, fanout=[2, 2])
    assert offs.tolist() == [0, 0, 0]
    p = u32(cs.csaw_walk(G, "degree", seeds, 5))
    assert p[0, 0] == iso and (p[:, 1:] == cs.NONE).all()
    # length 0 walk: just the seed
    assert u32(cs.csaw_walk(G, "degree", seeds, 0)).tolist() == [[iso], [iso]]


def test_errors(cfg1):
    G, og, g = cfg1
    bad = torch.tensor([0, 5000], dtype=torch.int32, device=DEV)
    with pytest.raises(cs.CsawError) as ei:
        cs.csaw_sample(G, "degree", bad, fanout=[2])
    assert ei.value.status == 2
    with pytest.raises(cs.CsawError):
        cs.csaw_sample(G, "node2vec", bad, fanout=[2])
    with pytest.raises(cs.CsawError) as ei:
        cs.csaw_graph_create(torch.tensor([0, 2, 1], device=DEV), torch.tensor([1, 0], dtype=torch.int32, device=DEV))
    assert ei.value.status == 3
    with pytest.raises(cs.CsawError) as ei:
        cs.csaw_graph_create(torch.tensor([0, 1, 2], device=DEV), torch.tensor([1, 7], dtype=torch.int32, device=DEV))
    assert ei.value.status == 3


def test_host_buffers_equal_device_buffers(cfg1):
    G, og, g = cfg1
    seeds_h = instance_seeds(g, 64)
    d = cs.csaw_sample(G, "degree", seeds_h.to(DEV), fanout=[2, 2], rng_seed=3)
    h = cs.csaw_sample(G, "degree", seeds_h.pin_memory(), fanout=[2, 2], rng_seed=3)
    for a, b in zip(d, h):
        assert torch.equal(a.cpu(), b)
    wd = cs.csaw_walk(G, "degree", seeds_h.to(DEV), 100, rng_seed=3)
    wh = cs.csaw_walk(G, "degree", seeds_h, 100, rng_seed=3)
    assert torch.equal(wd.cpu(), wh)


def test_sharding_by_instance_base(cfg1):
    """Determinism contract: shards [0,n/2) + [n/2,n) with instance_base == one run."""
    G, og, g = cfg1
    seeds = instance_seeds(g, 64).to(DEV)
    full = cs.csaw_sample(G, "degree", seeds, fanout=[2, 2], rng_seed=7)
    a = cs.csaw_sample(G, "degree", seeds[:32].contiguous(), fanout=[2, 2], rng_seed=7)
    b = cs.csaw_sample(G, "degree", seeds[32:].contiguous(), fanout=[2, 2], rng_seed=7, instance_base=32)
    assert torch.equal(full[2], torch.cat([a[2], b[2]]))
    wf = cs.csaw_walk(G, "degree", seeds, 64, rng_seed=7)
    wa = cs.csaw_walk(G, "degree", seeds[:40].contiguous(), 64, rng_seed=7)
    wb = cs.csaw_walk(G, "degree", seeds[40:].contiguous(), 64, rng_seed=7, instance_base=40)
    assert torch.equal(wf, torch.cat([wa, wb]))


def test_repeatable(cfg1):
    G, og, g = cfg1
    seeds = instance_seeds(g, 64).to(DEV)
    a = cs.csaw_walk(G, "degree", seeds, 300, rng_seed=1)
    b = cs.csaw_walk(G, "degree", seeds, 300, rng_seed=1)
    c = cs.csaw_walk(G, "degree", seeds, 300, rng_seed=2)
    assert torch.equal(a, b) and not torch.equal(a, c)


@pytest.mark.parametrize("m,n,L", [(2048, 5, 200), (2049, 4, 150), (33, 40, 300), (64, 7, 100), (1, 5000, 37)])
def test_mdrw_pool_sizes(medium, m, n, L):
    """k_mdrw_fast (pools <= 2,048 slots: register block totals, 16 B slot records) and
    k_mdrw (larger pools, or CSAW_GRAPH_MDRW_GENERIC) against the oracle, incl. ragged last
    blocks and more instances than resident warps."""
    G2, og2, g2 = medium
    s = mdrw_seeds(g2, n, m).numpy()
    e = check_mdrw(G2, og2, s, L, rng_seed=7, instances=range(0, n, max(1, n // 40)))
    for fl in (cs.CSAW_GRAPH_MDRW_GENERIC, cs.CSAW_GRAPH_MDRW_ALT_RECORDS):   # large-pool kernel; packed slot records
        Gv = cs.csaw_graph_create(g2.row_ptr.to(DEV), g2.col_idx.to(DEV), device=0, flags=fl)
        e2 = u32(cs.csaw_walk(Gv, cs.make_bias("mdrw", pool_size=m), torch.as_tensor(s.view(np.int32)).to(DEV), L,
                              rng_seed=7))
        Gv.close()
        assert np.array_equal(e, e2), hex(fl)


def test_mdrw_next_meta(medium):
    """CSAW_GRAPH_NEXT_META: the new pool vertex's row and degree come with the picked CSR
    entry (nmp); CSAW_GRAPH_NEXT_RECORD: entry, row and degree in one 16 B record (packed and
    16 B slot records) -- same edges as without them and as the oracle."""
    _, og2, g2 = medium
    Gm = cs.csaw_graph_create(g2.row_ptr.to(DEV), g2.col_idx.to(DEV), next_meta=True)
    assert Gm.info()["device_bytes"] >= 8 * g2.col_idx.numel()
    for m, n, L in [(2000, 6, 300), (37, 50, 200)]:
        s = mdrw_seeds(g2, n, m, set_id=3).numpy()
        e = check_mdrw(Gm, og2, s, L, rng_seed=17, instances=range(0, n, max(1, n // 10)))
        G0, _, _ = medium
        e0 = u32(cs.csaw_walk(G0, cs.make_bias("mdrw"), torch.as_tensor(s.view(np.int32)).to(DEV), L, rng_seed=17))
        assert np.array_equal(e, e0)
        for fl in (0, cs.CSAW_GRAPH_MDRW_ALT_RECORDS):   # 16 B next-vertex records (CSAW_GRAPH_NEXT_RECORD)
            Gr = cs.csaw_graph_create(g2.row_ptr.to(DEV), g2.col_idx.to(DEV), next_record=True, flags=fl)
            assert Gr.info()["device_bytes"] >= 16 * g2.col_idx.numel()
            er = u32(cs.csaw_walk(Gr, cs.make_bias("mdrw"), torch.as_tensor(s.view(np.int32)).to(DEV), L, rng_seed=17))
            Gr.close()
            assert np.array_equal(e, er), hex(fl)
    Gm.close()


@pytest.mark.parametrize("kind", ["degree", "uniform", "node2vec", "mdrw"])
def test_walk_into_pinned_host_output(medium, kind):
    """A pinned host `path` is written by the kernels directly (zero-copy); a pageable one is
    staged and copied.  Both must equal the device-buffer result."""
    G, og, g = medium
    if kind == "mdrw":
        seeds = mdrw_seeds(g, 40, 64)
        shape, L = (40, 90, 2), 90
    else:
        seeds = instance_seeds(g, 300, set_id=7)
        shape, L = (300, 91), 90
    b = cs.make_bias(kind, p=2.0, q=0.5)
    ref = cs.csaw_walk(G, b, seeds.to(DEV), L, rng_seed=3)
    pinned = torch.empty(shape, dtype=torch.int32).pin_memory()
    pageable = torch.empty(shape, dtype=torch.int32)
    cs.csaw_walk(G, b, seeds.pin_memory(), L, rng_seed=3, out=pinned)
    cs.csaw_walk(G, b, seeds, L, rng_seed=3, out=pageable)
    assert torch.equal(ref.cpu(), pinned) and torch.equal(ref.cpu(), pageable)


@pytest.mark.parametrize("kind", ["degree", "uniform", "node2vec", "mdrw"])
def test_walk_seed_out_of_range(medium, kind):
    """A seed >= V is rejected before any walk kernel reads a row (OUT_OF_RANGE)."""
    G, og, g = medium
    V = g.row_ptr.numel() - 1
    if kind == "mdrw":
        seeds = mdrw_seeds(g, 4, 8).clone()
        seeds[2, 5] = V
    else:
        seeds = instance_seeds(g, 40).clone()
        seeds[17] = V + 3
    for dev in (DEV, "cpu"):
        with pytest.raises(cs.CsawError) as ei:
            cs.csaw_walk(G, cs.make_bias(kind, p=2.0, q=0.5), seeds.to(dev), 20, rng_seed=1)
        assert ei.value.status == 2


@pytest.mark.parametrize("workload,fanout", [("degree", [2, 2]), ("layer", [2, 3]), ("forest_fire", []),
                                             ("degree", [40])])
def test_sample_into_pinned_host_output(cfg1, workload, fanout):
    """Pinned host outputs: the fused sampler's copy writes them directly (zero-copy); a
    fused-path fallback (fanout 40 > 32) stages through device scratch.  Both equal the
    device-buffer result."""
    G, og, g = cfg1
    seeds = instance_seeds(g, 200, set_id=9)
    kw = dict(fanout=fanout, depth=2, rng_seed=5, pf=0.7)
    ref = cs.csaw_sample(G, workload, seeds.to(DEV), **kw)
    cap = int(ref[1].numel()) + 16
    out = [torch.empty(seeds.numel() + 1, dtype=torch.int64).pin_memory(),
           torch.empty(cap, dtype=torch.int32).pin_memory(), torch.empty(cap, dtype=torch.int32).pin_memory(),
           torch.empty(cap, dtype=torch.uint8).pin_memory()]
    got = cs.csaw_sample(G, workload, seeds.pin_memory(), out=out, **kw)
    for a, b in zip(ref, got):
        assert torch.equal(a.cpu(), b.cpu())
