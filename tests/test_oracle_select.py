"""Pins for the oracle's selection without replacement (§4.2).

- Fig. 6(b)/(c) worked examples in integer form.
- Theorem 2 checked exhaustively: the BRS step equals ITS over the
  updated CTPS for every pre-selected s and every survivor position x'.
- The distribution of select_wor equals successive sampling ("updated
  sampling", Fig. 6(b)) by brute-force enumeration + chi-square.
"""
import itertools

import numpy as np
import pytest
from scipy import stats

import oracle as O
from tests._golden import paper_examples


def updated_its(b, taken, x2):
    """Fig. 6(b): rebuild the CTPS over survivors (excluding `taken`), search x2."""
    acc = 0
    for i, bi in enumerate(b):
        if i in taken or bi == 0:
            continue
        if x2 < acc + bi:
            return i
        acc += bi
    raise AssertionError("x2 outside survivor space")


def test_fig6b_updated_sampling_example():
    ex = paper_examples()["fig6b_updated_sampling"]
    S2 = O.prefix(ex["survivor_biases"])
    assert S2.tolist() == ex["S_prime"]
    assert np.round(S2 / S2[-1], 2).tolist() == ex["F_prime_2dp"]
    x = int(np.floor(ex["r"] * S2[-1]))           # 0.58 * 9 -> 5
    survivors = ["v5", "v9", "v10", "v11"]
    assert survivors[O.its(S2, x)] == ex["selected"]


def test_fig6c_brs_example_integer_and_float_forms():
    ex = paper_examples()["fig6c_brs"]
    b = paper_examples()["fig1b_ctps"]["biases"]
    cands = paper_examples()["fig1b_ctps"]["candidates"]
    # float form exactly as printed: r'/lambda = 0.58 * (1 - (h - l)) = 0.348; > l -> + delta
    lam = 1.0 / (1.0 - (ex["h"] - ex["l"]))
    r = ex["r_prime"] / lam
    assert abs(r - ex["r_adjusted"]) < 1e-12
    assert r > ex["l"]
    r2 = r + (ex["h"] - ex["l"])
    assert abs(r2 - ex["r_after_delta"]) < 1e-12
    F = O.prefix(b) / 15.0
    assert cands[int(np.searchsorted(F, r2, side="right") - 1)] == ex["selected"]
    # integer form: x' = floor(0.58 * (15 - 6)) = 5 >= l*T = 3 -> y = 11 -> v10
    x2 = int(np.floor(ex["r_prime"] * (15 - 6)))
    assert cands[O.brs_step(b, 1, x2)] == ex["selected"]
    # "identical as updated sampling"
    assert O.brs_step(b, 1, x2) == updated_its(b, {1}, x2)


def test_theorem2_exhaustive():
    """For every pre-selected s (b_s > 0) and every x' in [0, T - b_s):
    BRS(x') == ITS over the updated CTPS at x' (Theorem 2, Eq. 5-8)."""
    rng = np.random.default_rng(2009)
    cases = 0
    for _ in range(150):
        n = int(rng.integers(1, 14))
        b = rng.integers(0, 12, size=n).tolist()
        if rng.random() < 0.3:
            b[int(rng.integers(0, n))] = int(rng.integers(40, 200))   # a dominant bias
        T = sum(b)
        for s in range(n):
            if b[s] == 0 or T - b[s] == 0:
                continue
            for x2 in range(T - b[s]):
                assert O.brs_step(b, s, x2) == updated_its(b, {s}, x2)
                cases += 1
    assert cases > 10_000


def successive_probs(b, k):
    """Exact law of ordered k-tuples under successive sampling (updated
    sampling, Fig. 6(b); Theorem 1 applied to the survivors at every pick)."""
    T = sum(b)
    pos = [i for i, x in enumerate(b) if x > 0]
    probs = {}
    for tup in itertools.permutations(pos, k):
        p, rem = 1.0, T
        for s in tup:
            p *= b[s] / rem
            rem -= b[s]
        probs[tup] = p
    return probs


def chi2_pvalue(counts: dict, probs: dict, n: int):
    keys = list(probs.keys())
    exp = np.array([probs[k] * n for k in keys])
    obs = np.array([counts.get(k, 0) for k in keys], dtype=float)
    assert sum(counts.get(k, 0) for k in counts if k not in probs) == 0, "impossible outcome drawn"
    # merge categories with expected < 5 into one bin
    small = exp < 5
    if small.any():
        exp = np.append(exp[~small], exp[small].sum())
        obs = np.append(obs[~small], obs[small].sum())
    return stats.chisquare(obs, exp).pvalue


@pytest.mark.parametrize("b,k,a_max", [
    ([3, 6, 2, 2, 2], 2, 64),          # Fig. 1 pool
    ([3, 6, 2, 2, 2], 3, 64),
    ([90, 5, 3, 1, 1], 3, 64),         # skewed: frequent collisions
    ([1, 1, 1, 1, 50], 2, 64),
    ([0, 7, 0, 1, 3, 0, 2], 3, 64),    # zero-width regions
    ([1000, 1000, 1, 1, 1], 4, 2),     # attempt cap 2: the updated-sampling fallback fires
    ([90, 5, 3, 1, 1], 4, 2),
])
def test_select_wor_law_matches_successive_sampling(b, k, a_max):
    N = 24000
    counts = {}
    fallback_seen = False
    for inst in range(N):
        picks, att = O.select_wor(b, k, 0xC0FFEE, inst, 0, 0, a_max=a_max, with_attempts=True)
        assert len(picks) == k and len(set(picks)) == k
        assert all(b[s] > 0 for s in picks)
        fallback_seen |= att > 2 * k
        counts[tuple(picks)] = counts.get(tuple(picks), 0) + 1
    p = chi2_pvalue(counts, successive_probs(b, k), N)
    assert p > 1e-4, p
    if a_max == 2:
        assert fallback_seen


def test_select_wor_select_all_and_empty():
    # k >= #positive candidates: all of them, ascending (reading R8)
    assert O.select_wor([3, 0, 2, 5], 3, 1, 0, 0, 0) == [0, 2, 3]
    assert O.select_wor([3, 0, 2, 5], 10, 1, 0, 0, 0) == [0, 2, 3]
    assert O.select_wor([3, 0, 2, 5], 0, 1, 0, 0, 0) == []
    assert O.select_wor([0, 0], 1, 1, 0, 0, 0) == []
    assert O.select_wor([], 2, 1, 0, 0, 0) == []


def test_select_wor_deterministic_and_keyed():
    b = [5, 1, 9, 2, 2, 7, 1]
    a = O.select_wor(b, 3, 42, 7, 1, 99)
    assert a == O.select_wor(b, 3, 42, 7, 1, 99)
    # changing any key component changes the draw stream (with overwhelming probability
    # over a handful of alternatives)
    alts = {tuple(O.select_wor(b, 3, 42, 7 + d, 1, 99)) for d in range(1, 9)}
    assert len(alts | {tuple(a)}) > 1


def test_brs_fewer_attempts_than_repeated_sampling():
    """Fig. 11 direction: BRS needs fewer draws per pick than naive
    repeated sampling on a skewed pool.  Repeated sampling's expected draws for
    pick j are T / (T - taken mass); BRS uses at most 2 per round."""
    b = [90, 5, 3, 1, 1]
    k = 3
    N = 4000
    brs = 0
    for inst in range(N):
        _, att = O.select_wor(b, k, 7, inst, 0, 0, with_attempts=True)
        brs += att
    # expected repeated-sampling draws by enumeration of the successive law
    exp_rep = 0.0
    T = sum(b)
    for tup, p in successive_probs(b, k).items():
        taken = 0
        for s in tup:
            exp_rep += p * T / (T - taken)
            taken += b[s]
    assert brs / N < exp_rep


@pytest.mark.parametrize("mode", ["repeated", "updated"])
@pytest.mark.parametrize("b,k", [([3, 6, 2, 2, 2], 3), ([90, 5, 3, 1, 1], 3), ([0, 7, 0, 1, 3, 0, 2], 3)])
def test_baseline_migrations_have_the_same_law(mode, b, k):
    """Repeated sampling (Fig. 6(a)) and updated sampling (Fig. 6(b)) are the
    paper's baselines: same successive-sampling law, different draw usage."""
    O.set_migration(mode)
    try:
        N = 20000
        counts = {}
        draws = 0
        for inst in range(N):
            picks, att = O.select_wor(b, k, 99, inst, 0, 0, with_attempts=True)
            assert len(set(picks)) == k
            counts[tuple(picks)] = counts.get(tuple(picks), 0) + 1
            draws += att
        assert chi2_pvalue(counts, successive_probs(b, k), N) > 1e-4
        if mode == "updated":
            assert draws == N * k          # one draw per pick, never a collision
    finally:
        O.set_migration("brs")


def test_fig11_direction_brs_vs_repeated():
    """Fig. 11: BRS reduces the draws per pick vs repeated sampling."""
    b = [400, 40, 20, 10, 5, 5, 3, 1, 1]
    k = 4
    tot = {}
    for mode in ("brs", "repeated"):
        O.set_migration(mode)
        tot[mode] = sum(O.select_wor(b, k, 5, i, 0, 0, with_attempts=True)[1] for i in range(5000))
    O.set_migration("brs")
    assert tot["brs"] < tot["repeated"]
