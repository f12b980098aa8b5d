"""Narrow walk index (csrc/wix.cuh; NEXT-1 static-bias cache): degree-biased
walks searched through u32 fanout-128 nodes and FL-entry leaf blocks must be
bit-identical to the oracle for every leaf fanout, including rows deep enough for
three internal levels, and to the u64 index path (walk_index=False)."""

import numpy as np
import pytest
import torch

import paper_2009_09103_b200 as cs
from synth import instance_seeds, rmat_csr
from tests._golden import gtoy
from tests._parity import DEV, check_walk, u32

import oracle as O

pytestmark = pytest.mark.gpu

# (leaf fanout, lanes per walker: 32 = one warp per walker, 8 / 16 = sub-warp groups)
LEAVES = [(32, 32), (64, 32), (128, 32), (32, 8), (64, 8), (128, 8), (64, 16), (128, 16), (64, "nohead")]


def star_csr(V=700_001, d1=20_001):
    """Vertex 0 adjacent to 1..V-1 (d = 700000: three internal levels at leaf fanout 32,
    two at 128), vertex 1 to 2..d1, plus a ring over 1..V-1."""
    u = np.arange(1, V, dtype=np.int64)
    ring = np.stack([u, np.where(u + 1 < V, u + 1, 1)], 1)
    e = np.concatenate([np.stack([np.zeros_like(u), u], 1),
                        np.stack([np.ones(d1 - 1, np.int64), np.arange(2, d1 + 1, dtype=np.int64)], 1),
                        np.sort(ring, 1)])
    e = np.unique(e, axis=0)
    src = np.concatenate([e[:, 0], e[:, 1]])
    dst = np.concatenate([e[:, 1], e[:, 0]])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    rp = np.zeros(V + 1, np.int64)
    np.add.at(rp, src + 1, 1)
    return np.cumsum(rp), dst.astype(np.uint32)


def make(rp, col, leaf, walk_index=True):
    leaf, group = leaf if isinstance(leaf, tuple) else (leaf, 32)
    nohead = group == "nohead"   # (64, 32) walks the vertex heads (k_walk_head); this one the records
    group = 32 if nohead else group
    flags = ({128: 0, 64: cs.CSAW_GRAPH_WALK_LEAF_64, 32: cs.CSAW_GRAPH_WALK_LEAF_32}[leaf]
             | {32: 0, 16: cs.CSAW_GRAPH_WALK_GROUP_16, 8: cs.CSAW_GRAPH_WALK_GROUP_8}[group]
             | (cs.CSAW_GRAPH_WALK_NO_HEADS if nohead else 0))
    rpt = torch.as_tensor(np.asarray(rp, dtype=np.int64))
    ct = torch.as_tensor(np.asarray(col).astype(np.uint32).view(np.int32))
    G = cs.csaw_graph_create(rpt.to(DEV), ct.to(DEV), ctps_cache=True, walk_index=walk_index, flags=flags)
    assert G.info()["walk_index_leaf"] == (leaf if walk_index else 0)
    return G, O.Graph(rpt.numpy(), ct.numpy().view(np.uint32))


@pytest.fixture(scope="module")
def star():
    return star_csr()


@pytest.mark.parametrize("leaf", LEAVES)
def test_wix_rmat(leaf):
    g = rmat_csr(1 << 15, 1 << 19, 3)
    G, og = make(g.row_ptr, g.col_idx, leaf)
    seeds = instance_seeds(g, 300, set_id=2).numpy()
    check_walk(G, og, "degree", seeds, 257, rng_seed=9, instance_base=12345)
    st = cs.csaw_stats(G)
    assert st["pools"] > 0 and st["index_bytes"] >= 16 * st["pools"] and st["neighbours_scanned"] == 0
    G.close()


@pytest.mark.parametrize("leaf", LEAVES)
def test_wix_star_deep(star, leaf):
    G, og = make(*star, leaf)
    seeds = np.array([0, 1, 2, 699_999, 350_000, 0, 1, 20_000, 20_001, 7], dtype=np.uint32)
    check_walk(G, og, "degree", seeds, 64, rng_seed=3)
    G.close()


@pytest.mark.parametrize("leaf", [(32, 32), (32, 8), (128, 8), (64, 16)])
def test_wix_gtoy_and_tail(leaf):
    rp, col = gtoy()
    G, og = make(rp, col, leaf)
    seeds = np.tile(np.arange(12, dtype=np.uint32), 40)   # 480 walkers: several per warp slot
    check_walk(G, og, "degree", seeds, 70, rng_seed=5)     # length not a multiple of 32
    check_walk(G, og, "degree", seeds[:1], 1, rng_seed=6)
    check_walk(G, og, "degree", seeds[:3], 0, rng_seed=6)
    G.close()


@pytest.mark.parametrize("n,length,leaf", [(2000, 300, (64, 8)), (2001, 301, (64, 32)), (50_003, 41, (64, 8)),
                                           (40_001, 33, (128, 16))])
def test_wix_equals_u64_index(n, length, leaf):
    """Ragged walker counts (not a multiple of the group count) and more walkers than
    resident groups (grid-stride rounds) against the u64 index path."""
    g = rmat_csr(1 << 16, 1 << 20, 7)
    seeds = torch.as_tensor(instance_seeds(g, n, set_id=1).numpy().view(np.int32)).to(DEV)
    G1, _ = make(g.row_ptr, g.col_idx, leaf)
    G2, _ = make(g.row_ptr, g.col_idx, 64, walk_index=False)
    p1 = u32(cs.csaw_walk(G1, cs.make_bias("degree"), seeds, length, rng_seed=21))
    p2 = u32(cs.csaw_walk(G2, cs.make_bias("degree"), seeds, length, rng_seed=21))
    assert np.array_equal(p1, p2)
    G1.close()
    G2.close()


def test_wix_isolated_seed():
    # seed with degree 0 and a walker reaching a vertex whose neighbours all have degree 0 is
    # impossible in a symmetric graph; a directed toy graph covers T == 0 (walk ends, R20)
    rp = np.array([0, 2, 2, 3, 3], np.int64)          # 0 -> {1, 3}; 1 isolated; 2 -> {1}; 3 none
    col = np.array([1, 3, 1], np.uint32)
    for leaf in LEAVES:
        G, og = make(rp, col, leaf)
        check_walk(G, og, "degree", np.array([0, 1, 2, 3], np.uint32), 5, rng_seed=1)
        G.close()


def boundary_csr():
    """Rows at the vertex-head boundaries: d = 7,936 (top level of 124 entries, inline),
    7,937 / 8,100 / 8,192 (125 / 127 / 128 top entries: read from the node array), d = 60
    (inline leaf) and 61..64 (leaf read from the leaf arrays), plus a ring."""
    V = 9_000
    adj = {v: set() for v in range(V)}

    def link(a, b):
        if a != b:
            adj[a].add(b)
            adj[b].add(a)

    for hub, d in [(0, 7936), (1, 7937), (2, 8100), (3, 8192)]:
        for u in range(10, 10 + d):
            link(hub, u % V if u < V else 10 + (u % (V - 10)))
    for v, d in [(4, 60), (5, 61), (6, 62), (7, 63), (8, 64)]:
        for u in range(100 + 97 * v, 100 + 97 * v + d):
            link(v, u)
    for v in range(9, V):
        link(v, v + 1 if v + 1 < V else 9)
    rp = np.zeros(V + 1, np.int64)
    rp[1:] = np.cumsum([len(adj[v]) for v in range(V)])
    col = np.concatenate([np.array(sorted(adj[v]), np.uint32) for v in range(V)])
    return rp, col


@pytest.mark.parametrize("leaf", [(128, 32), (64, 32), (64, "nohead"), (32, 32)])
def test_wix_head_boundaries(leaf):
    rp, col = boundary_csr()
    deg = np.diff(rp)
    assert {7936, 7937, 8192, 60, 61, 64} <= set(deg[:9].tolist())
    G, og = make(rp, col, leaf)
    seeds = np.array([0, 1, 2, 3, 4, 5, 6, 7, 8] * 8 + [100, 500, 4000], dtype=np.uint32)
    check_walk(G, og, "degree", seeds, 120, rng_seed=31)
    G.close()
