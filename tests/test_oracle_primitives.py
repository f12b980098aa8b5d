"""Pins for the oracle's primitives: Philox KATs, below(), CTPS prefix, ITS.

Every expected value comes from the paper (cited), a published KAT, or a closed
form -- never from the oracle itself or the CUDA path.
"""
import numpy as np
import pytest

import oracle as O
from tests._golden import paper_examples, philox_kats


@pytest.mark.parametrize("ctr,key,out", philox_kats())
def test_philox_known_answers(ctr, key, out):
    # Random123 kat_vectors (tests/golden/philox_kat.txt)
    assert O.philox4x32_10(ctr, key) == out


def test_below_closed_forms():
    M = 12345
    assert O.below(0, M) == 0
    assert O.below(2**64 - 1, M) == M - 1          # floor((2^64-1) M / 2^64) = M-1
    assert O.below(2**63, M) == M // 2             # exactly half
    assert O.below(2**62, 4) == 1                  # quarter of 4
    assert O.below(2**64 - 1, 1) == 0              # M = 1 has one outcome
    # the value k is produced exactly by U in [ceil(k 2^64/M), ceil((k+1) 2^64/M))
    for k in (0, 1, 77, M - 1):
        lo = -(-(k << 64) // M)
        hi = -(-((k + 1) << 64) // M) - 1
        assert O.below(lo, M) == k and O.below(hi, M) == k
        if lo > 0:
            assert O.below(lo - 1, M) == k - 1


def test_fig1b_ctps_and_its():
    ex = paper_examples()["fig1b_ctps"]          # Fig. 1(b)
    S = O.prefix(ex["biases"])
    assert S.tolist() == ex["S"]
    T = int(S[-1])
    F = np.round(S.astype(float) / T, 2).tolist()
    assert F == ex["F_2dp"]
    x = int(np.floor(ex["r"] * T))                 # r = 0.5 -> x = 7 in [0, 15)
    s = O.its(S, x)
    assert ex["candidates"][s] == ex["selected"]   # v7


def test_its_uniform_is_identity():
    # unit biases: S_i = i, so the region of x is x itself (closed form)
    S = O.prefix([1] * 37)
    for x in range(37):
        assert O.its(S, x) == x


def test_its_zero_width_regions_never_chosen():
    b = [0, 5, 0, 0, 3, 0]
    S = O.prefix(b)
    got = [O.its(S, x) for x in range(int(S[-1]))]
    assert got == [1] * 5 + [4] * 3


def test_its_region_sizes_equal_biases():
    # Theorem 1: |{x : its(x) = k}| / T = b_k / sum(b)
    rng = np.random.default_rng(5)
    for _ in range(20):
        b = rng.integers(0, 9, size=rng.integers(1, 12)).tolist()
        if sum(b) == 0:
            continue
        S = O.prefix(b)
        counts = np.bincount([O.its(S, x) for x in range(int(S[-1]))], minlength=len(b))
        assert counts.tolist() == b


def test_ff_theta_matches_paper_pf():
    # P_f = 0.7; theta = floor(0.7 * 2^32) computed on the binary64 value of 0.7
    assert O.ff_theta(0.7) == 0xB3333333
    assert O.ff_theta(0.0) == 0
    assert O.ff_theta(0.5) == 2**31


def test_n2v_scale():
    # p = 2, q = 0.5 (config 3): alpha in {1/2, 1, 2} -> m = 2 gives {1, 2, 4}
    assert O.n2v_scale(2.0, 0.5) == 2
    assert O.n2v_scale(1.0, 1.0) == 1
    assert O.n2v_scale(4.0, 0.25) == 4
    import math
    assert O.n2v_scale(math.pi, math.e) == 0      # no integral scale -> float path
