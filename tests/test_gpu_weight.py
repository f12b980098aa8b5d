"""GPU parity of the per-edge bias streams (vscan.cuh) against the oracle.

- CSAW_BIAS_WEIGHT (EdgeBias = w(e), Eq. 3) is the float path (R28): every GPU
  transition is checked against the oracle's step at the GPU's own vertex (teacher forcing);
  a pick may differ only where the oracle's draw lies within 1e-6 * T of a CTPS boundary
  (north star).  Sampling instances are compared whole and excused only under the same rule.
- The materialised degree bias (CSAW_GRAPH_EDGE_BIAS) is integer: bit-exact.
- The walker-group width G (warps sharing one pool) never changes a result (R7).
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import edge_weights, instance_seeds, rmat_csr
from tests._parity import DEV, check_sample, check_walk, u32
from tests.test_gpu_parity import hub_csr

pytestmark = pytest.mark.gpu
TOL = 1e-6


def wgraph(rp, col, w, **kw):
    rp_t = torch.as_tensor(np.asarray(rp, dtype=np.int64))
    c_t = torch.as_tensor(np.asarray(col).astype(np.uint32).view(np.int32))
    w_t = torch.as_tensor(np.asarray(w, dtype=np.float32))
    G = cs.csaw_graph_create(rp_t.to(DEV), c_t.to(DEV), device=0, weights=w_t.to(DEV), **kw)
    return G, O.Graph(rp_t.numpy(), c_t.numpy().view(np.uint32), w_t.numpy())


@pytest.fixture(scope="module")
def cfg1w():
    g = rmat_csr(1024, 16384, 1)
    w = edge_weights(g, 1, zero_frac=0.1)
    G, og = wgraph(g.row_ptr.numpy(), g.col_idx.numpy(), w.numpy())
    return G, og, g


@pytest.fixture(scope="module")
def mediumw():
    g = rmat_csr(1 << 15, 1 << 19, 7)
    w = edge_weights(g, 3, zero_frac=0.05)
    G, og = wgraph(g.row_ptr.numpy(), g.col_idx.numpy(), w.numpy(), edge_bias=True)
    return G, og, g


@pytest.fixture(scope="module")
def hubw():
    rp, col = hub_csr()
    src = np.repeat(np.arange(rp.size - 1), np.diff(rp))
    h = (src * 2654435761 + col.astype(np.int64) * 40503) % 1000
    w = ((h + 1) / 64.0).astype(np.float32)
    w[h < 30] = 0.0
    G, og = wgraph(rp, col, w, edge_bias=True)
    return G, og, rp


def weight_walk_check(G, og, seeds, length, rng_seed, walkers=None):
    s = torch.as_tensor(np.asarray(seeds).astype(np.uint32).view(np.int32)).to(DEV)
    path = u32(cs.csaw_walk(G, cs.make_bias("weight"), s, length, rng_seed=rng_seed))
    excused = 0
    for w in (range(len(seeds)) if walkers is None else walkers):
        assert path[w][0] == seeds[w]
        for t in range(length):
            v = int(path[w][t])
            if v == O.NONE32:
                assert path[w][t + 1] == O.NONE32
                continue
            ref, mg = O.weight_walk_step(og, v, w, t, rng_seed)
            if int(path[w][t + 1]) != ref:
                assert mg <= TOL, f"walker {w} step {t}: gpu {path[w][t + 1]} oracle {ref} margin {mg}"
                excused += 1
    return path, excused


@pytest.mark.parametrize("rng_seed", [1, 2])
def test_weight_walk_cfg1(cfg1w, rng_seed):
    G, og, g = cfg1w
    seeds = instance_seeds(g, 300).numpy().view(np.uint32)
    _, excused = weight_walk_check(G, og, seeds, 120, rng_seed)
    assert excused <= 2


def test_weight_walk_medium_and_group_invariance(mediumw):
    G, og, g = mediumw
    seeds = instance_seeds(g, 6000).numpy().view(np.uint32)   # >= 32 per SM: one warp per walker
    full, excused = weight_walk_check(G, og, seeds, 64, 5, walkers=range(0, 6000, 25))
    assert excused <= 2
    # 16 walkers: 8-warp groups share each pool -- same bits for the same walkers
    s16 = torch.as_tensor(seeds[:16].view(np.int32)).to(DEV)
    few = u32(cs.csaw_walk(G, cs.make_bias("weight"), s16, 64, rng_seed=5))
    assert np.array_equal(few, full[:16])


def test_weight_walk_hub(hubw):
    G, og, _ = hubw
    seeds = np.array([0, 1, 0, 2, 1, 0, 7, 0], np.uint32)   # d = 300,000 and 20,001 pools
    _, excused = weight_walk_check(G, og, seeds, 40, 9)
    assert excused <= 1


def test_weight_walk_zero_weight_row_ends():
    rp = np.array([0, 2, 3, 4], np.int64)
    col = np.array([1, 2, 0, 0], np.uint32)
    w = np.array([0.0, 0.0, 1.0, 1.0], np.float32)
    G, og = wgraph(rp, col, w)
    s = torch.tensor([1, 0], dtype=torch.int32, device=DEV)
    path = u32(cs.csaw_walk(G, cs.make_bias("weight"), s, 4, rng_seed=1))
    assert path[0].tolist() == [1, 0] + [O.NONE32] * 3
    assert path[1].tolist() == [0] + [O.NONE32] * 4


def weight_sample_check(G, og, seeds, fanout, rng_seed):
    s = torch.as_tensor(np.asarray(seeds).astype(np.uint32).view(np.int32)).to(DEV)
    offs, src, dst, dep = cs.csaw_sample(G, cs.make_bias("weight"), s, fanout=fanout, rng_seed=rng_seed)
    offs = offs.cpu().numpy().astype(np.int64)
    src, dst, dep = u32(src), u32(dst), dep.cpu().numpy()
    excused = 0
    for i, sv in enumerate(seeds):
        es, ed, ee, mg = O.weight_sample(og, fanout, len(fanout), int(sv), i, rng_seed)
        a, b = int(offs[i]), int(offs[i + 1])
        same = b - a == es.size and np.array_equal(src[a:b], es) and np.array_equal(dst[a:b], ed) \
            and np.array_equal(dep[a:b], ee)
        if not same:
            assert mg <= TOL, f"instance {i}: differs from the oracle, margin {mg}"
            excused += 1
    return excused


@pytest.mark.parametrize("fanout", [[2, 2], [5, 3], [1]])
def test_weight_sampling_cfg1(cfg1w, fanout):
    G, og, g = cfg1w
    seeds = instance_seeds(g, 256).numpy().view(np.uint32)
    assert weight_sample_check(G, og, seeds, fanout, 3) <= 2


def test_weight_sampling_batched_and_multipass(hubw):
    G, og, _ = hubw
    # fanout 40 > 32: the batched driver with picks beyond lane 31 (glist); collisions on hubs
    seeds = np.array([0, 1, 5, 0, 1], np.uint32)
    assert weight_sample_check(G, og, seeds, [40, 2], 4) <= 1
    assert weight_sample_check(G, og, seeds, [3, 3], 6) <= 1


def test_weight_sampling_batched_flag(cfg1w):
    _, og, g = cfg1w
    w = torch.as_tensor(og.w)
    Gb = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV), device=0, weights=w.to(DEV), batched_only=True)
    seeds = instance_seeds(g, 128).numpy().view(np.uint32)
    assert weight_sample_check(Gb, og, seeds, [2, 2], 7) <= 2


# ---------------------------------------------------------------- materialised degree bias (integer, exact)
def test_edge_bias_degree_walk_exact(mediumw):
    G, og, g = mediumw
    assert G.info()["edge_bias"] == 1 and G.info()["ctps_cache"] == 0
    seeds = instance_seeds(g, 5000).numpy().view(np.uint32)
    check_walk(G, og, "degree", seeds, 80, rng_seed=2, walkers=range(0, 5000, 20))
    # few walkers: 8-warp groups, still bit-exact
    check_walk(G, og, "degree", seeds[:12], 80, rng_seed=2)


def test_edge_bias_hub_exact(hubw):
    G, og, _ = hubw
    check_walk(G, og, "degree", np.array([0, 1, 3, 0], np.uint32), 50, rng_seed=11)


def test_integer_weights_equal_the_degree_walk(mediumw):
    """w(e) = deg(col[e]) as fp32: the float stream picks what the exact integer walk picks
    (up to boundary draws)."""
    _, og, g = mediumw
    deg = (g.row_ptr[1:] - g.row_ptr[:-1])
    wd = deg[g.col_idx.long()].to(torch.float32)
    G = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV), device=0, weights=wd.to(DEV))
    seeds = instance_seeds(g, 400).numpy().view(np.uint32)
    s = torch.as_tensor(seeds.view(np.int32)).to(DEV)
    pw = u32(cs.csaw_walk(G, cs.make_bias("weight"), s, 50, rng_seed=3))
    pd = u32(cs.csaw_walk(G, cs.make_bias("degree"), s, 50, rng_seed=3))
    assert (pw != pd).any(axis=1).sum() <= 2


def test_weight_errors(cfg1w):
    _, og, g = cfg1w
    rp, col = g.row_ptr.to(DEV), g.col_idx.to(DEV)
    bad = torch.as_tensor(og.w).clone()
    bad[17] = -1.0
    with pytest.raises(cs.CsawError) as e:
        cs.csaw_graph_create(rp, col, device=0, weights=bad.to(DEV))
    assert e.value.status == 3
    bad[17] = float("nan")
    with pytest.raises(cs.CsawError) as e:
        cs.csaw_graph_create(rp, col, device=0, weights=bad.to(DEV))
    assert e.value.status == 3
    G0 = cs.csaw_graph_create(rp, col, device=0)
    s = torch.tensor([1, 2], dtype=torch.int32, device=DEV)
    with pytest.raises(cs.CsawError) as e:
        cs.csaw_walk(G0, cs.make_bias("weight"), s, 4)
    assert e.value.status == 1
    with pytest.raises(cs.CsawError) as e:
        cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, weights=torch.as_tensor(og.w), budget_bytes=1 << 20)
    assert e.value.status == 8


# ---------------------------------------------------------------- weighted node2vec (R33)
def test_weighted_node2vec_teacher_forced(mediumw):
    """node2vec on a weighted graph: b = alpha * w(e), float path; every GPU transition
    equals the oracle's step at the GPU's own (prev, v) unless the draw is within 1e-6 of a
    boundary.  Integer-scale p, q (2, 0.5) take the float path too once the graph has weights."""
    G, og, g = mediumw
    seeds = instance_seeds(g, 600).numpy().view(np.uint32)
    s = torch.as_tensor(seeds.view(np.int32)).to(DEV)
    for p, q in ((2.0, 0.5), (np.pi, np.e)):
        path = u32(cs.csaw_walk(G, cs.make_bias("node2vec", p=p, q=q), s, 30, rng_seed=12))
        excused = 0
        for w in range(0, 600, 3):
            for t in range(30):
                v = int(path[w][t])
                if v == O.NONE32:
                    assert path[w][t + 1] == O.NONE32
                    continue
                prev = O.NONE32 if t == 0 else int(path[w][t - 1])
                ref, mg = O.node2vec_w_step(og, p, q, prev, v, w, t, 12)
                if int(path[w][t + 1]) != ref:
                    assert mg <= TOL, (p, q, w, t, mg)
                    excused += 1
        assert excused <= 2


def test_weighted_node2vec_p1q1_equals_weight_walk(mediumw):
    G, og, g = mediumw
    s = instance_seeds(g, 256).to(DEV)
    a = cs.csaw_walk(G, cs.make_bias("node2vec", p=1.0, q=1.0), s, 40, rng_seed=2)
    b = cs.csaw_walk(G, cs.make_bias("weight"), s, 40, rng_seed=2)
    # both are the edge-weight walk (b = 1.0f * w); the kernels sum in different orders, so
    # they may differ only at boundary draws
    assert (a != b).any(dim=1).sum().item() <= 2
