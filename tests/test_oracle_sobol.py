"""Pins for oracle steps O1-O3 (direction numbers, randomisation, Sobol' integers).

Each pin is external to the oracle: NVIDIA's libcurand host generator (the
paper's generator), the published Joe-Kuo rows, SPEC.md's hand
traces of the P:166 recurrence, the defining properties of primitive
polynomials and of digital (0,m,1)-nets (stratification).
"""
import os

import numpy as np
import pytest

from tests import _curand

HERE = os.path.dirname(os.path.abspath(__file__))
need_curand = pytest.mark.skipif(not _curand.available(), reason="libcurand not present")


def test_recurrence_spec_examples(O):
    import ctypes
    # poly x^3+x+1 (c1=0, c2=1 -> a=0b01), initial (1,3,7) -> m4 = (4*3)^(8*1)^1 = 5
    m_init = np.array([1, 3, 7], np.uint32)
    out = np.zeros(4, np.uint64)
    rc = O.lib().or_expand_recurrence(3, 1, m_init.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), 4,
                                      out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    assert rc == 0 and int(out[3]) == 5
    # poly x+1 (q=1), initial (1) -> m2 = 2*1 ^ 1 = 3
    m_init = np.array([1], np.uint32)
    out = np.zeros(2, np.uint64)
    O.lib().or_expand_recurrence(1, 0, m_init.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), 2,
                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    assert int(out[1]) == 3


def test_joe_kuo_published_rows(O):
    rows = [l.split() for l in open(os.path.join(HERE, "golden", "joe_kuo_rows.txt")) if not l.startswith("#")]
    for r in rows:
        dim, s, a = int(r[0]), int(r[1]), int(r[2])
        assert O.polynomial(dim - 1) == (s, a)
        m = [int(x) for x in r[3:]]
        v = O.direction_numbers(dim)[dim - 1]
        assert [int(v[b]) >> (31 - b) for b in range(s)] == m


def test_direction_numbers_invariants(O):
    # every m_k odd and < 2^k; g_k in (0,1); dimension 1 is the identity
    v = O.direction_numbers(1024)
    assert all(int(v[0][b]) == 1 << (31 - b) for b in range(32))
    for j in range(1024):
        for b in range(32):
            m = int(v[j][b]) >> (31 - b)
            assert m & 1 and m < (1 << (b + 1))


def _polymulmod(a, b, f, deg):
    r = 0
    while b:
        if b & 1:
            r ^= a
        b >>= 1
        a <<= 1
        if a >> deg & 1:
            a ^= f
    return r


def _polypowmod(e, f, deg):
    result, base = 1, 2  # polynomial "x"
    while e:
        if e & 1:
            result = _polymulmod(result, base, f, deg)
        base = _polymulmod(base, base, f, deg)
        e >>= 1
    return result


def _prime_factors(n):
    out, p = set(), 2
    while p * p <= n:
        while n % p == 0:
            out.add(p)
            n //= p
        p += 1
    if n > 1:
        out.add(n)
    return out


def test_polynomials_are_primitive_and_distinct(O):
    # cannot be factored, and the smallest p with poly | x^p + 1 is 2^q - 1.
    seen = set()
    for j in range(1, 1024):
        s, a = O.polynomial(j)
        f = (1 << s) | (a << 1) | 1
        assert f not in seen
        seen.add(f)
        n = (1 << s) - 1
        if s == 1:
            assert f == 0b11
            continue
        assert _polypowmod(n, f, s) == 1
        for q in _prime_factors(n):
            assert _polypowmod(n // q, f, s) != 1


@need_curand
def test_direction_numbers_match_curand_joekuo6(O):
    assert np.array_equal(O.direction_numbers(1024), _curand.direction_vectors(False, 1024))


@need_curand
def test_plain_sobol_matches_curand_host_generator(O):
    # Gray-code order with point 0 included, dimension-major output
    d, n = 64, 4096
    ref = _curand.host_generate(_curand.QUASI_SOBOL32, n, d)
    got = O.sobol_u32(0, 0, d, 0, n, O.config(randomization=O.RAND_NONE))
    assert np.array_equal(got, ref)


@need_curand
def test_scrambled_sobol_formula_matches_curand(O):
    # y = c ^ XOR_{b in gray(k)} v'_b with cuRAND's scrambled vectors and constants
    d, n = 64, 4096
    ref = _curand.host_generate(_curand.QUASI_SCRAMBLED_SOBOL32, n, d)
    v = _curand.direction_vectors(True, d)
    c = _curand.scramble_constants(d)
    assert np.array_equal(O.sobol_from_vectors(v, c, 0, d, 0, n), ref)


@need_curand
def test_philox_matches_curand_host(O):
    ref = _curand.host_generate(_curand.PSEUDO_PHILOX4_32_10, 4, 1, seed=1234)[0]
    assert np.array_equal(O.philox([0, 0, 0, 0], [1234, 0]), ref)


def test_philox_known_answers(O):
    for line in open(os.path.join(HERE, "golden", "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        assert O.philox(w[0:4], w[4:6]).tolist() == w[6:10]


@pytest.mark.parametrize("mode", [0, 1])
def test_randomised_points_stay_dyadic_nets(O, mode):
    # A left-matrix scramble + digital shift is a bijection on every elementary
    # interval: each aligned block of 2^m points has exactly one point in each
    # [i 2^-m, (i+1) 2^-m).
    m, d = 10, 64
    for rep in (0, 7):
        y = O.sobol_u32(rep, 0, d, 0, 3 << m, O.config(randomization=mode))
        for blk in range(3):
            top = y[:, blk << m:(blk + 1) << m] >> (32 - m)
            for j in range(d):
                assert np.array_equal(np.sort(top[j]), np.arange(1 << m))


def test_lms_scramble_is_nontrivial_and_replicate_dependent(O):
    plain, _ = O.randomization(O.DEFAULT_SEED, 0, 8, O.RAND_NONE)
    v0, c0 = O.randomization(O.DEFAULT_SEED, 0, 8, O.RAND_LMS_SHIFT)
    v1, c1 = O.randomization(O.DEFAULT_SEED, 1, 8, O.RAND_LMS_SHIFT)
    assert not np.array_equal(plain, v0) and not np.array_equal(v0, v1) and not np.array_equal(c0, c1)
    # L is lower-triangular with unit diagonal in MSB-first digit order, so the
    # first nonzero digit of every direction number is preserved: v'_b and v_b
    # have the same bit length; and L stays invertible (v'_b remain independent).
    for j in range(8):
        for b in range(32):
            assert int(v0[j][b]).bit_length() == int(plain[j][b]).bit_length()


def test_randomised_point_uniform_over_replicates(O):
    # fixed (dim, k), the replicate ensemble is uniform: chi-square on 64 bins at 0.001
    from scipy import stats
    R = 4096
    vals = np.array([O.sobol_u32(rep, 5, 6, 3, 4)[0, 0] for rep in range(R)])
    counts = np.bincount(vals >> 26, minlength=64)
    chi2 = ((counts - R / 64) ** 2 / (R / 64)).sum()
    assert stats.chi2.sf(chi2, 63) > 1e-3
