"""Pins of the oracle's nested (Owen) scrambling, O2b (SURVEY.md row f4,
DESIGN.md reading 27).  Each test checks a property every nested uniform scramble
must have, independent of the hash that draws the permutations:

  * nesting: digit i of the output depends only on digits 0..i-1 and digit i of
    the input (points sharing a prefix keep it, and split at the same digit);
  * bijectivity of every prefix map (here the 2^16 16-digit prefixes);
  * uniformity over seeds (each output digit is a fair coin for a fixed input);
  * scrambled Sobol' points keep the (t, m, s)-net structure (1-D stratification
    and the t = 0 two-dimensional elementary boxes of dimensions 0 and 1);
  * the variance rate: for a smooth 1-D integrand, Owen-scrambled nets have
    Var = O(N^-3) (Owen 1997), a digital shift alone only O(N^-2).
"""
import numpy as np

import oracle as O

RNG = np.random.default_rng(20221018)


def digit(y, i):  # digit i of a 32-bit coordinate, MSB first
    return (y >> (31 - i)) & 1


def test_nesting_prefix_kept_and_first_difference_kept():
    for _ in range(3000):
        seed = int(RNG.integers(0, 2**32))
        p = int(RNG.integers(0, 32))
        y1 = int(RNG.integers(0, 2**32))
        y2 = y1 ^ (1 << (31 - p))                           # flip digit p ...
        if p < 31:
            y2 ^= int(RNG.integers(0, 2 ** (31 - p)))       # ... and randomise the digits after it
        s1, s2 = O.owen_scramble(y1, seed), O.owen_scramble(y2, seed)
        mask = (0xFFFFFFFF << (32 - p)) & 0xFFFFFFFF if p else 0
        assert (s1 & mask) == (s2 & mask)                   # shared prefix stays shared
        assert digit(s1, p) != digit(s2, p)                 # and they still split at digit p


def test_prefix_map_is_a_bijection():
    for seed in (0, 1, 0xDEADBEEF, int(RNG.integers(0, 2**32))):
        tops = set()
        for pre in range(1 << 16):
            low = int(RNG.integers(0, 1 << 16))
            tops.add(O.owen_scramble((pre << 16) | low, seed) >> 16)
        assert len(tops) == 1 << 16


def test_each_output_digit_is_a_fair_coin_over_seeds():
    n = 4000
    for y in (0, 0x80000000, 0x12345678, 0xFFFFFFFF):
        outs = np.array([O.owen_scramble(y, int(s)) for s in RNG.integers(0, 2**32, n)], np.uint64)
        for i in range(32):
            f = float(np.mean((outs >> np.uint64(31 - i)) & np.uint64(1)))
            assert abs(f - 0.5) < 5 * 0.5 / np.sqrt(n), (y, i, f)


def test_scrambled_sobol_keeps_the_net_structure():
    m = 10
    cfg = O.config(randomization=O.RAND_OWEN, seed=77)
    for rep in (0, 3):
        y = O.sobol_u32(rep, 0, 8, 0, 1 << m, cfg).astype(np.uint64)
        plain = O.sobol_u32(rep, 0, 8, 0, 1 << m, O.config(randomization=O.RAND_NONE)).astype(np.uint64)
        assert not np.array_equal(y, plain)
        for j in range(8):                                  # (0, m, 1)-net in every dimension
            assert len(set((y[j] >> np.uint64(32 - m)).tolist())) == 1 << m
        for a in range(m + 1):                              # dims 0, 1: t = 0 -> one point per 2^a x 2^(m-a) box
            b = m - a
            box = ((y[0] >> np.uint64(32 - a)) << np.uint64(b)) | (y[1] >> np.uint64(32 - b))
            assert len(set(box.tolist())) == 1 << m, (rep, a)


def _rqmc_var(randomization, m, L=256):
    cfg = O.config(randomization=randomization, seed=5)
    est = []
    for rep in range(L):
        y = O.sobol_u32(rep, 0, 1, 0, 1 << m, cfg)[0].astype(np.float64)
        u = (y + 0.5) * 2.0**-32
        est.append(np.mean(np.exp(u)))
    return np.var(est)


def test_variance_rate_is_cubic_for_owen_and_quadratic_for_a_shift():
    r_owen = _rqmc_var(O.RAND_OWEN, 5) / _rqmc_var(O.RAND_OWEN, 9)      # 16x points
    r_shift = _rqmc_var(O.RAND_SHIFT, 5) / _rqmc_var(O.RAND_SHIFT, 9)
    assert r_owen > 16**2.6, r_owen            # ~16^3 = 4096
    assert r_shift < 16**2.4, r_shift          # ~16^2 = 256
