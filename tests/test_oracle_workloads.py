"""Pins for the oracle's five workloads on G_toy and small R-MAT graphs.

Exact laws are enumerated by brute force from the paper's definitions
(Theorem 1 per pick, successive sampling without replacement, UPDATE
post-filter) and compared by chi-square; exact special cases (node2vec
p=q=1 == simple walk, MDRW with one pool slot == simple walk, P_f = 0) and
invariants cover the rest.
"""
import itertools
import math

import numpy as np
import pytest
from scipy import stats

import oracle as O
from synth import rmat_csr, instance_seeds
from tests._golden import gtoy, paper_examples


@pytest.fixture(scope="module")
def G():
    rp, col = gtoy()
    return O.Graph(rp, col)


@pytest.fixture(scope="module")
def R():
    g = rmat_csr(1024, 16384, 1)          # config-1 graph
    return O.Graph.from_torch(g), g


def chi2(counts, probs, n):
    assert set(counts) <= set(probs), set(counts) - set(probs)
    keys = list(probs)
    exp = np.array([probs[k] * n for k in keys])
    obs = np.array([counts.get(k, 0) for k in keys], float)
    small = exp < 5
    if small.any():
        exp = np.append(exp[~small], exp[small].sum())
        obs = np.append(obs[~small], obs[small].sum())
    return stats.chisquare(obs, exp).pvalue


def successive(b, k):
    """ordered-tuple law of k picks without replacement (Fig. 6(b) semantics)."""
    pos = [i for i, x in enumerate(b) if x > 0]
    if k >= len(pos):
        return {tuple(pos): 1.0}
    T = sum(b)
    out = {}
    for tup in itertools.permutations(pos, k):
        p, rem = 1.0, T
        for s in tup:
            p *= b[s] / rem
            rem -= b[s]
        out[tup] = p
    return out


# ------------------------------------------------------------- neighbor sampling
def ns_law(G, seed, fanout, bias):
    """Exact law of the edge set of one neighbor-sampling instance (Fig. 2(b)
    main loop, Update = visited post-filter).  Enumerates every branch."""
    def pools(v):
        nb = G.nbrs(v).tolist()
        b = [G.deg(u) if bias == "degree" else 1 for u in nb]
        return nb, b

    law = {}

    def rec(d, F, visited, edges, p):
        if d == len(fanout) or not F:
            key = tuple(sorted(edges, key=lambda e: (e[2], e[0], e[1])))
            law[key] = law.get(key, 0.0) + p
            return
        # each frontier vertex independently; product over vertices
        branches = [((), 1.0)]
        for v in sorted(F):
            nb, b = pools(v)
            nxt = []
            for tup, q in successive(b, fanout[d]).items():
                picked = tuple(sorted(nb[s] for s in tup))
                for prev, pp in branches:
                    nxt.append((prev + ((v, picked),), pp * q))
            branches = nxt
        merged = {}
        for br, q in branches:
            merged[br] = merged.get(br, 0.0) + q
        for br, q in merged.items():
            new_edges = list(edges)
            nxtF = set()
            for v, picked in br:
                for u in picked:
                    new_edges.append((v, u, d + 1))
                    if u not in visited:
                        nxtF.add(u)
            rec(d + 1, nxtF, visited | nxtF, new_edges, p * q)

    rec(0, {seed}, {seed}, [], 1.0)
    return law


def edges_key(s, d, e):
    return tuple((int(a), int(b), int(c)) for a, b, c in zip(s, d, e))


def test_fig1_first_pick_law(G):
    """From v8 with bias = degree, one pick: (3,6,2,2,2)/15 (Fig. 1 caption
    P:127 + Theorem 1)."""
    N = 30000
    counts = {}
    for inst in range(N):
        s, d, e = O.neighbor_sample(G, O.KIND_DEGREE, [1], 1, 8, inst, 11)
        counts[int(d[0])] = counts.get(int(d[0]), 0) + 1
    probs = {5: 3 / 15, 7: 6 / 15, 9: 2 / 15, 10: 2 / 15, 11: 2 / 15}
    assert chi2(counts, probs, N) > 1e-4


@pytest.mark.parametrize("seed,fanout,bias", [(8, [2, 2], "degree"), (7, [2, 2], "degree"),
                                              (4, [2, 1], "uniform"), (8, [3], "degree")])
def test_neighbor_sampling_exact_law(G, seed, fanout, bias):
    law = ns_law(G, seed, fanout, bias)
    assert abs(sum(law.values()) - 1) < 1e-9
    N = 20000
    counts = {}
    kind = O.KIND_DEGREE if bias == "degree" else O.KIND_UNIFORM
    for inst in range(N):
        k = edges_key(*O.neighbor_sample(G, kind, fanout, len(fanout), seed, inst, 1234))
        counts[k] = counts.get(k, 0) + 1
    assert chi2(counts, law, N) > 1e-4


def test_neighbor_sampling_invariants(R):
    og, tg = R
    seeds = instance_seeds(tg, 64).numpy().astype(np.uint32)
    for i, sd in enumerate(seeds):
        s, d, e = O.neighbor_sample(og, O.KIND_DEGREE, [2, 2], 2, int(sd), i, 1)
        assert list(zip(e, s, d)) == sorted(zip(e, s, d))            # canonical order (R11)
        pairs = set()
        visited = {int(sd)}
        for a, b, c in zip(s, d, e):
            assert int(b) in set(og.nbrs(int(a)).tolist())          # edge exists
            assert (a, b) not in pairs                              # no duplicate edge
            pairs.add((a, b))
            assert 1 <= c <= 2
        # depth-1 sources are the seed; count = min(k, deg) on a symmetric graph
        d1 = [(a, b) for a, b, c in zip(s, d, e) if c == 1]
        assert all(a == sd for a, _ in d1) and len(d1) == min(2, og.deg(int(sd)))
        f1 = sorted({int(b) for _, b in d1} - visited)
        srcs2 = sorted({int(a) for a, b, c in zip(s, d, e) if c == 2})
        assert srcs2 == [v for v in f1 if og.deg(v) > 0]
        for v in f1:
            assert sum(1 for a, b, c in zip(s, d, e) if c == 2 and a == v) == min(2, og.deg(v))


def test_forest_fire_pf_zero_and_burn_law(G):
    # P_f = 0: nothing burns, no edges
    s, d, e = O.neighbor_sample(G, O.KIND_FF, [], 2, 8, 0, 5, pf=0.0)
    assert len(s) == 0
    # burn count law: P(x = n) = (1-th) th^n for n < deg, th^deg at n = deg (R15)
    th = O.ff_theta(0.7) / 2**32
    deg = 5
    probs = {n: (1 - th) * th ** n for n in range(deg)}
    probs[deg] = th ** deg
    N = 40000
    counts = {}
    for inst in range(N):
        x = O.ff_burn(99, inst, 0, 8, deg, 0.7)
        counts[x] = counts.get(x, 0) + 1
    assert chi2(counts, probs, N) > 1e-4


def test_forest_fire_law_one_level(G):
    """depth 1 from v8: burn x, then x uniform distinct neighbours."""
    th = O.ff_theta(0.7) / 2**32
    nb = G.nbrs(8).tolist()
    law = {}
    for x in range(len(nb) + 1):
        px = (1 - th) * th ** x if x < len(nb) else th ** len(nb)
        for combo in itertools.combinations(nb, x):
            key = tuple((8, u, 1) for u in combo)
            law[key] = law.get(key, 0) + px / math.comb(len(nb), x)
    N = 30000
    counts = {}
    for inst in range(N):
        k = edges_key(*O.neighbor_sample(G, O.KIND_FF, [], 1, 8, inst, 77, pf=0.7))
        counts[k] = counts.get(k, 0) + 1
    assert chi2(counts, law, N) > 1e-4


# ------------------------------------------------------------- layer sampling
def layer_law(G, seed, fanout):
    law = {}

    def rec(d, F, visited, edges, p):
        if d == len(fanout) or not F:
            key = tuple(sorted(edges, key=lambda e: (e[2], e[0], e[1])))
            law[key] = law.get(key, 0.0) + p
            return
        pool = [(v, u) for v in sorted(F) for u in G.nbrs(v).tolist()]   # union, canonical order
        b = [G.deg(u) for _, u in pool]
        for tup, q in successive(b, fanout[d]).items():
            new_edges = list(edges)
            nxt = set()
            for s in tup:
                v, u = pool[s]
                new_edges.append((v, u, d + 1))
                if u not in visited:
                    nxt.add(u)
            rec(d + 1, nxt, visited | nxt, new_edges, p * q)

    rec(0, {seed}, {seed}, [], 1.0)
    return law


@pytest.mark.parametrize("seed,fanout", [(8, [2, 2]), (7, [1, 3]), (4, [2, 2])])
def test_layer_sampling_exact_law(G, seed, fanout):
    law = layer_law(G, seed, fanout)
    N = 20000
    counts = {}
    for inst in range(N):
        k = edges_key(*O.layer_sample(G, fanout, len(fanout), seed, inst, 4321))
        counts[k] = counts.get(k, 0) + 1
    assert chi2(counts, law, N) > 1e-4


# ------------------------------------------------------------- walks
def test_degree_walk_transition_law(G):
    N = 20000
    for v in (8, 7, 4):
        nb = G.nbrs(v).tolist()
        T = sum(G.deg(u) for u in nb)
        probs = {u: G.deg(u) / T for u in nb}
        counts = {}
        for inst in range(N):
            u = O.walk_step(G, O.KIND_DEGREE, v, inst, 3, 55)
            counts[u] = counts.get(u, 0) + 1
        assert chi2(counts, probs, N) > 1e-4


def test_walks_are_valid_paths(R):
    og, tg = R
    seeds = instance_seeds(tg, 16).numpy().astype(np.uint32)
    for kind in (O.KIND_DEGREE, O.KIND_UNIFORM):
        for i, s0 in enumerate(seeds):
            p = O.walk(og, kind, 200, int(s0), i, 3)
            assert p[0] == s0 and p.size == 201
            for t in range(200):
                assert int(p[t + 1]) in set(og.nbrs(int(p[t])).tolist())


def test_degree_walk_stationary_law(G):
    """Reversible chain with edge weight deg(v) deg(u): pi(v) ∝ deg(v) Σ_{u∈N(v)} deg(u)."""
    w = np.array([G.deg(v) * sum(G.deg(u) for u in G.nbrs(v)) for v in range(G.V)], float)
    pi = w / w.sum()
    counts = np.zeros(G.V)
    for inst in range(400):
        p = O.walk(G, O.KIND_DEGREE, 500, 8, inst, 9)
        np.add.at(counts, p[100:].astype(np.int64), 1)      # after burn-in
    freq = counts / counts.sum()
    assert np.abs(freq - pi).sum() / 2 < 0.02


def test_node2vec_p1_q1_equals_simple_walk(R):
    """b ≡ const => below(U, c d) // c == below(U, d): identical paths (exact)."""
    og, tg = R
    seeds = instance_seeds(tg, 12).numpy().astype(np.uint32)
    for i, s0 in enumerate(seeds):
        a = O.node2vec(og, 1.0, 1.0, 60, int(s0), i, 17)
        b = O.walk(og, O.KIND_UNIFORM, 60, int(s0), i, 17)
        assert a.tolist() == b.tolist()


@pytest.mark.parametrize("p,q", [(2.0, 0.5), (math.pi, math.e)])
def test_node2vec_step_law(G, p, q):
    """prev = 9, v = 8 on G_toy: N(8) = [5,7,9,10,11], N(9) = [8,10]:
    alpha = 1/p for u = 9, 1 for u = 10 (∈ N(9)), 1/q otherwise.
    (p, q) = (pi, e) exercises the float path (fp32 biases, fp64 sums)."""
    alpha = {5: 1 / q, 7: 1 / q, 9: 1 / p, 10: 1.0, 11: 1 / q}
    Z = sum(alpha.values())
    probs = {u: a / Z for u, a in alpha.items()}
    N = 30000
    counts = {}
    for inst in range(N):
        u, mg = O.node2vec_step(G, p, q, 9, 8, inst, 1, 808)
        counts[u] = counts.get(u, 0) + 1
        assert 0 <= mg <= 1
    assert chi2(counts, probs, N) > 1e-4


def test_node2vec_first_step_uniform(G):
    N = 20000
    counts = {}
    for inst in range(N):
        p = O.node2vec(G, 2.0, 0.5, 1, 8, inst, 3)
        counts[int(p[1])] = counts.get(int(p[1]), 0) + 1
    assert chi2(counts, {u: 0.2 for u in [5, 7, 9, 10, 11]}, N) > 1e-4


# ------------------------------------------------------------- MDRW
def test_mdrw_single_slot_equals_simple_walk(R):
    """m = 1: the VertexBias pick is always slot 0 and the EdgeBias draw is the
    simple walk's draw U(i, t, 0, EDGE) -> identical sequences (exact)."""
    og, tg = R
    seeds = instance_seeds(tg, 10).numpy().astype(np.uint32)
    for i, s0 in enumerate(seeds):
        e = O.mdrw(og, [int(s0)], 80, i, 21)
        w = O.walk(og, O.KIND_UNIFORM, 80, int(s0), i, 21)
        assert e[:, 0].tolist() == w[:-1].tolist()
        assert e[:, 1].tolist() == w[1:].tolist()


def test_fig4_mdrw_vertex_bias(G):
    """Fig. 4: pool {v8, v0, v3}, VertexBias = degree -> P(v8) = 5/8;
    EdgeBias = 1 -> uniform neighbour; Update replaces v8's slot."""
    ex = paper_examples()["fig4_mdrw"]
    N = 24000
    counts, nb_counts = {}, {}
    for inst in range(N):
        e = O.mdrw(G, ex["pool"], 1, inst, 31)
        v, u = int(e[0, 0]), int(e[0, 1])
        counts[v] = counts.get(v, 0) + 1
        if v == ex["picked"]:
            nb_counts[u] = nb_counts.get(u, 0) + 1
    assert chi2(counts, {8: 5 / 8, 0: 1 / 8, 3: 2 / 8}, N) > 1e-4
    n8 = counts[8]
    assert chi2(nb_counts, {u: 0.2 for u in G.nbrs(8).tolist()}, n8) > 1e-4
    assert ex["neighbor"] in nb_counts


def test_mdrw_update_replaces_slot(G):
    e = O.mdrw(G, [8, 0, 3], 50, 5, 1)
    pool = [8, 0, 3]
    for t in range(50):
        v, u = int(e[t, 0]), int(e[t, 1])
        assert v in pool and u in G.nbrs(v).tolist()
        pool[pool.index(v)] = u            # in-place slot replacement (R18)


# ------------------------------------------------------------- OOM facts
def test_fig8_partition_facts():
    ex = paper_examples()["fig8_oom"]
    b = O.partition_bounds(12, ex["partitions"])
    assert b == [0, 4, 8, 12]
    assert O.active_counts(b, ex["seeds"]) == ex["active_counts"]
    assert O.partition_bounds(10, 3) == [0, 4, 7, 10]      # remainder to the lowest (R23)
    rp, col = gtoy()
    G = O.Graph(rp, col)
    for a, c in ex["edges_present"]:
        assert c in G.nbrs(a).tolist()


# ------------------------------------------------------------- Table-1 walk variants (NEXT-3)
def test_mh_walk_acceptance_law(G):
    """MH walk: from v=0 (deg 1) the only proposal is 7 (deg 6): accept 1/6, else stay."""
    N = 24000
    counts = {}
    for inst in range(N):
        u = O.walk_variant_step(G, O.KIND_MH, 0.0, 0, 0, inst, 2, 31)
        counts[u] = counts.get(u, 0) + 1
    assert chi2(counts, {7: 1 / 6, 0: 5 / 6}, N) > 1e-4


def test_mh_walk_stationary_uniform(G):
    """MH with acceptance min(1, d(v)/d(u)) has the uniform stationary law."""
    counts = np.zeros(G.V)
    for inst in range(300):
        p = O.walk_variant(G, O.KIND_MH, 600, 8, inst, 4)
        np.add.at(counts, p[100:].astype(np.int64), 1)
    freq = counts / counts.sum()
    assert np.abs(freq - 1 / G.V).sum() / 2 < 0.03


def test_restart_and_jump_with_zero_probability_are_the_simple_walk(R):
    og, tg = R
    seeds = instance_seeds(tg, 8).numpy().astype(np.uint32)
    for i, s0 in enumerate(seeds):
        w = O.walk(og, O.KIND_UNIFORM, 50, int(s0), i, 9)
        assert O.walk_variant(og, O.KIND_RESTART, 50, int(s0), i, 9, 0.0).tolist() == w.tolist()
        assert O.walk_variant(og, O.KIND_JUMP, 50, int(s0), i, 9, 0.0).tolist() == w.tolist()


def test_restart_probability(G):
    """Restart: from v=8 (0 not a neighbour) P(next = s0 = 0) = floor(pr 2^32) / 2^32."""
    pr = 0.3
    th = np.floor(pr * 2**32) / 2**32
    N = 30000
    back = sum(O.walk_variant_step(G, O.KIND_RESTART, pr, 0, 8, inst, 5, 77) == 0 for inst in range(N))
    assert chi2({1: back, 0: N - back}, {1: th, 0: 1 - th}, N) > 1e-4


def test_jump_law(G):
    """Jump: from v=0 (N = {7}): 7 w.p. (1-th) + th/12, every other vertex th/12."""
    pr = 0.25
    th = np.floor(pr * 2**32) / 2**32
    probs = {u: th / 12 for u in range(12)}
    probs[7] += 1 - th
    N = 40000
    counts = {}
    for inst in range(N):
        u = O.walk_variant_step(G, O.KIND_JUMP, pr, 0, 0, inst, 1, 5)
        counts[u] = counts.get(u, 0) + 1
    assert chi2(counts, probs, N) > 1e-4


def _bfs_ball_edges(og, seed, depth):
    """Snowball sampling written out as a plain BFS: every edge out of
    every vertex first reached at distance < depth, tagged with its distance + 1."""
    dist = {seed: 0}
    layer = [seed]
    out = []
    for d in range(depth):
        nxt = []
        for v in layer:
            for u in og.nbrs(v).tolist():
                out.append((d + 1, v, int(u)))
                if u not in dist:
                    dist[u] = d + 1
                    nxt.append(int(u))
        layer = nxt
    return sorted(out)


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_snowball_is_the_bfs_ball(G, R, depth):
    """NEXT-3 snowball = select-all neighbor sampling; pinned to a BFS written here."""
    og, tg = R
    cases = [(G, v) for v in range(G.V) if G.deg(v) > 0]
    cases += [(og, int(s)) for s in instance_seeds(tg, 6).numpy()]
    for i, (g, sd) in enumerate(cases):
        s, d, e = O.neighbor_sample(g, O.KIND_SNOWBALL, [], depth, sd, i, 3)
        got = sorted(zip(e.tolist(), s.tolist(), d.tolist()))
        assert got == _bfs_ball_edges(g, sd, depth)
        # no draws: independent of the RNG seed and instance id
        s2, d2, e2 = O.neighbor_sample(g, O.KIND_SNOWBALL, [], depth, sd, i + 7, 11)
        assert np.array_equal(s, s2) and np.array_equal(d, d2) and np.array_equal(e, e2)
