"""Pins of the oracle's edge-weight (EdgeBias = w(e), Eq. 3) float path (R28).

Nothing here re-types the oracle's formulas.  The float path is pinned by:
- the paper's Fig. 1(b) worked example with the biases as fp32 weights;
- reduction to hand-pinned primitives: k = 1 equals the hand-pinned single draw
  (tests/test_oracle_float.py), and integer-valued weights w(e) = deg(col[e])
  reproduce the exact-integer degree-biased oracle (a different arithmetic: below()
  on u64 vs r * T in fp64) wherever the draw is not within 1e-6 of a boundary;
- the successive-sampling law by brute-force enumeration + chi-square
  (Theorem 1 on the survivors, Fig. 6(b)), including zero weights and the
  updated-sampling fallback (a_max = 2);
- the walk's transition law (Theorem 1: P(u) = w(v,u) / sum_w) by chi-square.
"""
import numpy as np
import pytest

import oracle as O
from synth import edge_weights, instance_seeds, rmat_csr
from tests._golden import paper_examples
from tests.test_oracle_select import chi2_pvalue, successive_probs

TWO53 = 1 << 53


def U_of(k):
    return (k << 11) | 0x5A5


def philox_U(inst, t=0, slot=0, j=0, a=0, seed=1):
    o = O.philox4x32_10([inst, t, slot, (j << 14) | a], [seed & 0xFFFFFFFF, seed >> 32])
    return o[0] | (o[1] << 32)


def test_fig1b_float_weights():
    ex = paper_examples()["fig1b_ctps"]
    b = np.array(ex["biases"], dtype=np.float32)
    s, mg = O.select_float(b, U_of(int(ex["r"] * TWO53)))       # x = 0.5 * 15 = 7.5 in [3, 9)
    assert ex["candidates"][s] == ex["selected"]
    assert mg == pytest.approx(1.5 / 15)                          # nearest boundary S_2 = 9


def test_k1_equals_the_single_draw():
    rng = np.random.default_rng(5)
    for inst in range(300):
        n = int(rng.integers(1, 12))
        b = rng.random(n).astype(np.float32) * (rng.random(n) > 0.2)
        if b.sum() == 0:
            continue
        picks, mg = O.select_wor_float(b, 1, 9, inst, 2, 77)
        s, mg1 = O.select_float(b, philox_U(inst, 2, 77, seed=9))
        if (b > 0).sum() == 1:
            assert picks == [int(np.flatnonzero(b)[0])]
            continue
        assert picks == [s] and mg == mg1


@pytest.mark.parametrize("b,k,a_max", [
    ([3.0, 6.0, 2.0, 2.0, 2.0], 2, 64),
    ([0.25, 1.5, 0.0, 7.75, 0.5], 3, 64),
    ([90.5, 5.25, 3.0, 1.0, 0.125], 3, 64),       # skewed: collisions migrate
    ([1000.0, 999.5, 1.0, 1.0, 1.0], 4, 2),       # a_max 2: exact updated-sampling fallback
])
def test_select_wor_float_law(b, k, a_max):
    N = 24000
    counts = {}
    for inst in range(N):
        picks, _ = O.select_wor_float(b, k, 0xBEEF, inst, 1, 3, a_max=a_max)
        assert len(set(picks)) == k and all(b[s] > 0 for s in picks)
        counts[tuple(picks)] = counts.get(tuple(picks), 0) + 1
    assert chi2_pvalue(counts, successive_probs(b, k), N) > 1e-4


def test_select_wor_float_select_all_and_empty():
    assert O.select_wor_float([3.0, 0.0, 2.0, 5.0], 3, 1, 0, 0, 0)[0] == [0, 2, 3]
    assert O.select_wor_float([3.0, 0.0, 2.0, 5.0], 9, 1, 0, 0, 0)[0] == [0, 2, 3]
    assert O.select_wor_float([0.0, 0.0], 1, 1, 0, 0, 0)[0] == []


def test_integer_weights_reproduce_the_integer_selection():
    """fp32 integer biases through the float path == oracle_select_wor (exact integers,
    below()) for the same Philox counters, except draws within 1e-6 of a boundary."""
    rng = np.random.default_rng(11)
    same = excused = 0
    for inst in range(3000):
        n = int(rng.integers(2, 40))
        b = rng.integers(0, 50, size=n)
        if rng.random() < 0.3:
            b[int(rng.integers(0, n))] = int(rng.integers(500, 5000))
        k = int(rng.integers(1, 6))
        pf, mg = O.select_wor_float(b.astype(np.float32), k, 3, inst, 0, 5)
        pi = O.select_wor(b.tolist(), k, 3, inst, 0, 5)
        if pf == pi:
            same += 1
        else:
            assert mg <= 1e-6, (b, k, pf, pi, mg)
            excused += 1
    assert same >= 2990


@pytest.fixture(scope="module")
def R():
    g = rmat_csr(1024, 16384, 1)
    deg = (g.row_ptr[1:] - g.row_ptr[:-1]).numpy()
    wdeg = deg[g.col_idx.numpy()].astype(np.float32)     # w(e) = deg(col[e])
    return g, O.Graph.from_torch(g), wdeg


def test_degree_weights_reproduce_the_degree_walk(R):
    g, og, wdeg = R
    ow = O.Graph(og.row_ptr, og.col, wdeg)
    seeds = instance_seeds(g, 64).numpy()
    for i, s in enumerate(seeds):
        pw, mg = O.weight_walk(ow, 60, int(s), i, 4, with_margins=True)
        pd = O.walk(og, O.KIND_DEGREE, 60, int(s), i, 4)
        if not np.array_equal(pw, pd):
            t = int(np.flatnonzero(pw != pd)[0]) - 1
            assert mg[t] <= 1e-6


def test_degree_weights_reproduce_degree_sampling(R):
    g, og, wdeg = R
    ow = O.Graph(og.row_ptr, og.col, wdeg)
    seeds = instance_seeds(g, 64).numpy()
    for i, s in enumerate(seeds):
        s1, d1, e1, mg = O.weight_sample(ow, [3, 2], 2, int(s), i, 8)
        s2, d2, e2 = O.neighbor_sample(og, O.KIND_DEGREE, [3, 2], 2, int(s), i, 8)
        if not (np.array_equal(s1, s2) and np.array_equal(d1, d2) and np.array_equal(e1, e2)):
            assert mg <= 1e-6


def test_weight_walk_transition_law():
    # v = 0 with neighbours 1..4 of weights (0.5, 0, 2.5, 1): P = (1/8, 0, 5/8, 2/8)
    rp = np.array([0, 4, 5, 6, 7, 8], np.int64)
    col = np.array([1, 2, 3, 4, 0, 0, 0, 0], np.uint32)
    w = np.array([0.5, 0.0, 2.5, 1.0, 1, 1, 1, 1], np.float32)
    og = O.Graph(rp, col, w)
    N = 16000
    cnt = np.zeros(5)
    for i in range(N):
        u, _ = O.weight_walk_step(og, 0, i, 3, 21)
        cnt[u] += 1
    assert cnt[0] == 0 and cnt[2] == 0
    exp = np.array([0.5, 2.5, 1.0]) / 4.0 * N
    from scipy import stats
    assert stats.chisquare(cnt[[1, 3, 4]], exp).pvalue > 1e-4


def test_zero_weight_rows_end_the_walk():
    rp = np.array([0, 2, 3, 4], np.int64)
    col = np.array([1, 2, 0, 0], np.uint32)
    w = np.array([0.0, 0.0, 1.0, 1.0], np.float32)
    path = O.weight_walk(O.Graph(rp, col, w), 5, 1, 0, 1)
    assert path[0] == 1 and path[1] == 0 and all(p == O.NONE32 for p in path[2:])


def test_weights_generator_is_symmetric_and_exact():
    g = rmat_csr(1024, 16384, 1)
    w = edge_weights(g, 1, 0.1).numpy()
    rp, col = g.row_ptr.numpy(), g.col_idx.numpy()
    src = np.repeat(np.arange(1024), np.diff(rp))
    d = dict(zip(zip(src.tolist(), col.tolist()), w.tolist()))
    assert all(d[(b, a)] == x for (a, b), x in d.items())
    assert 0.05 < (w == 0).mean() < 0.15 and np.isfinite(w).all() and (w >= 0).all()


# ---------------------------------------------------------------- weighted node2vec (R33)
def test_node2vec_w_with_p_q_1_is_the_weight_walk(R):
    """alpha = 1 everywhere (p = q = 1): b = 1.0f * w = w exactly, and step 0 is the weighted
    step -- the weighted node2vec walk is the edge-weight walk, pick for pick and margin for margin."""
    g, og, _ = R
    w = edge_weights(g, 5, zero_frac=0.05).numpy()
    ow = O.Graph(og.row_ptr, og.col, w)
    for i, s in enumerate(instance_seeds(g, 40).numpy()):
        a, ma = O.node2vec_w(ow, 1.0, 1.0, 40, int(s), i, 9, with_margins=True)
        b, mb = O.weight_walk(ow, 40, int(s), i, 9, with_margins=True)
        assert np.array_equal(a, b) and np.array_equal(ma, mb)


def test_node2vec_w_with_unit_weights_is_the_float_node2vec(R):
    """w = 1: b = alpha exactly, so every step after the first equals the (unweighted) float
    node2vec step at the same (prev, v) -- the pinned alpha law."""
    g, og, _ = R
    ow = O.Graph(og.row_ptr, og.col, np.ones(og.col.size, np.float32))
    p, q = np.pi, np.e
    for i, s in enumerate(instance_seeds(g, 30).numpy()):
        path = O.node2vec_w(ow, p, q, 30, int(s), i, 4)
        for t in range(1, 30):
            if path[t + 1] == O.NONE32:
                break
            u, _ = O.node2vec_step(og, p, q, int(path[t - 1]), int(path[t]), i, t, 4)
            assert u == path[t + 1]


def test_node2vec_w_transition_law():
    """v = 0 with prev = 1; N(0) = {1, 2, 3, 4}, N(1) = {0, 2}: alpha = (1/p, 1, 1/q, 1/q) for
    u = 1, 2, 3, 4; weights (2, 1, 0.5, 0) -> P proportional to (2/p, 1, 0.5/q, 0)."""
    rp = np.array([0, 4, 6, 7, 8, 9], np.int64)
    col = np.array([1, 2, 3, 4, 0, 2, 0, 0, 0], np.uint32)
    w = np.array([2.0, 1.0, 0.5, 0.0, 1.0, 1.0, 1.0, 1.0, 1.0], np.float32)
    og = O.Graph(rp, col, w)
    p, q = 2.0, 0.5
    N = 16000
    cnt = np.zeros(5)
    for i in range(N):
        u, _ = O.node2vec_w_step(og, p, q, 1, 0, i, 1, 33)
        cnt[u] += 1
    assert cnt[4] == 0 and cnt[0] == 0
    pr = np.array([2 / p, 1.0, 0.5 / q])
    from scipy import stats
    assert stats.chisquare(cnt[[1, 2, 3]], pr / pr.sum() * N).pvalue > 1e-4
