"""Pins of the oracle's float-bias selection (R28; the north star's 1e-6 boundary rule).

The draw U is an input here, so each case places x = r * T by hand:
r = (U >> 11) * 2^-53, i.e. U = k << 11 gives r = k / 2^53 exactly.  Expected
picks and margins are computed by hand from the definition
  s = max{i : S_i <= x, b_i > 0},  margin = min_{0<i<n} |x - S_i| / T,
not by re-running the oracle's formula.
"""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.filterwarnings("ignore")

TWO53 = 1 << 53


def U_of(k):
    """the 64-bit draw whose 53-bit fraction is k / 2^53"""
    return (k << 11) | 0x7FF          # the dropped low 11 bits must not matter


def test_draw_exactly_on_a_boundary():
    # b = (1, 1, 2): S = (0, 1, 2, 4), T = 4.  r = 1/2 -> x = 2.0 = S_2 exactly:
    # the region [S_2, S_3) holds x, so s = 2 and the margin is 0.
    s, mg = O.select_float([1.0, 1.0, 2.0], U_of(TWO53 // 2))
    assert s == 2 and mg == 0.0


def test_one_ulp_below_and_above_the_boundary():
    # r = 1/2 - 2^-53 -> x = 2 - 2^-51 (exact in binary64): still in [S_1, S_2) -> s = 1;
    # distance to S_2 is 2^-51, relative to T = 4: 2^-53.
    s, mg = O.select_float([1.0, 1.0, 2.0], U_of(TWO53 // 2 - 1))
    assert s == 1 and mg == 2.0 ** -53
    s, mg = O.select_float([1.0, 1.0, 2.0], U_of(TWO53 // 2 + 1))
    assert s == 2 and mg == 2.0 ** -53


def test_margin_is_relative_to_T_not_n():
    # x = 0.375 * 4 = 1.5: nearest interior boundaries S_1 = 1, S_2 = 2 at distance 0.5;
    # margin = 0.5 / T = 0.125 (a /n normalisation would give 0.1667).
    s, mg = O.select_float([1.0, 1.0, 2.0], U_of(3 * TWO53 // 8))
    assert s == 1 and mg == 0.125
    # b = (5, 5, 10, 20): T = 40, r = 0.3 -> x = 12 -> s = 2 ([10, 20)); margin = 2 / 40
    k = int(0.3 * TWO53)
    x = (k / TWO53) * 40.0
    s, mg = O.select_float([5.0, 5.0, 10.0, 20.0], U_of(k))
    assert s == 2 and mg == pytest.approx(abs(x - 10.0) / 40.0, rel=1e-12)


def test_end_boundaries_do_not_count_and_zero_weights_are_skipped():
    # x = 0 lies on S_0 = 0, which is not an interior boundary: margin = 1 / 4 (to S_1)
    s, mg = O.select_float([1.0, 1.0, 2.0], U_of(0))
    assert s == 0 and mg == 0.25
    # b = (1, 0, 1): S = (0, 1, 1, 2); x = 1.0 -> [S_2, S_3), never the zero-width region 1
    s, mg = O.select_float([1.0, 0.0, 1.0], U_of(TWO53 // 2))
    assert s == 2 and mg == 0.0
    # trailing zero weight: the last positive region takes the top of the range
    s, _ = O.select_float([1.0, 1.0, 0.0], U_of(TWO53 - 1))
    assert s == 1
    assert O.select_float([0.0, 0.0], U_of(5))[0] == -1


def test_fp32_biases_summed_in_fp64_left_to_right():
    # b = (2^24, 1, 1) as fp32: an fp32 running sum would stay at 2^24 (1 is lost),
    # fp64 keeps S = (0, 2^24, 2^24 + 1, 2^24 + 2).  x = r * T with r just above
    # (2^24 + 1) / T must pick s = 2.
    T = 2.0 ** 24 + 2
    k = math.ceil((2.0 ** 24 + 1) / T * TWO53)
    s, _ = O.select_float(np.array([2 ** 24, 1, 1], dtype=np.float32), U_of(k))
    assert s == 2


def test_frequencies_follow_the_biases():
    # Theorem 1: P(s) = b_s / T; 20,000 Philox draws (the oracle's own generator)
    b = np.array([0.5, 1.5, 3.0, 0.0, 5.0], dtype=np.float32)
    cnt = np.zeros(b.size)
    for i in range(20000):
        o = O.philox4x32_10([i, 7, 0, 0], [11, 0])
        s, _ = O.select_float(b, o[0] | (o[1] << 32))
        cnt[s] += 1
    p = b / b.sum()
    m = p > 0
    chi2 = float((((cnt - 20000 * p) ** 2)[m] / (20000 * p[m])).sum())
    assert cnt[3] == 0 and chi2 < 16.3        # chi-square, 3 dof, p ~ 0.001
