"""Pins for oracle step O4 (uniform lattice -> standard normal).

External references: mpmath at 40 digits (independent arbitrary-precision
erfinv) and scipy.special.ndtri (Cephes).  The lattice is u = (y + 1/2) 2^-32
(cuRAND's convention, PAPER.md:440 generator).
"""
import mpmath as mp
import numpy as np
from scipy.special import ndtri

mp.mp.dps = 40


def _exact(y):
    u = (mp.mpf(int(y)) + mp.mpf("0.5")) / mp.mpf(2) ** 32
    return float(-mp.sqrt(2) * mp.erfinv(1 - 2 * u))


def _ulp(x):
    return np.spacing(abs(x))


def test_pinned_values(O):
    # SURVEY.md B5 values, recomputed here with mpmath
    assert abs(O.normal_from_u32(0) - _exact(0)) <= _ulp(6.34)
    assert abs(O.normal_from_u32(0) - (-6.3379577545537892525)) <= 2 * _ulp(6.34)
    x = O.normal_from_u32(2 ** 31 - 1)
    assert abs(x - (-2.9180993729166226723e-10)) <= 2 * _ulp(x)
    # 0.975 -> 1.959964
    assert abs(O.inv_normal_cdf(0.975) - 1.959964) < 1e-6
    assert O.inv_normal_cdf(0.5) == 0.0


def test_against_mpmath_on_lattice(O):
    rng = np.random.default_rng(1)
    ys = np.concatenate([rng.integers(0, 2 ** 32, 3000, dtype=np.uint64),
                         np.arange(0, 200, dtype=np.uint64),                       # deep lower tail
                         2 ** 31 - 1 - np.arange(0, 200, dtype=np.uint64),         # around u = 1/2
                         2 ** 32 - 1 - np.arange(0, 100, dtype=np.uint64),         # deep upper tail
                         (rng.integers(0, 2 ** 22, 500, dtype=np.uint64))])       # tail region u < 1e-3
    worst = 0.0
    for y in ys:
        got, ref = O.normal_from_u32(int(y)), _exact(int(y))
        worst = max(worst, abs(got - ref) / _ulp(ref))
    assert worst <= 2.0, worst


def test_against_scipy_dense(O):
    rng = np.random.default_rng(2)
    ys = rng.integers(0, 2 ** 32, 200000, dtype=np.uint64)
    got = np.array([O.normal_from_u32(int(y)) for y in ys])
    ref = ndtri((ys.astype(np.float64) + 0.5) * 2.0 ** -32)
    assert np.max(np.abs(got - ref) / np.maximum(np.spacing(np.abs(ref)), 1e-300)) < 8


def test_exact_mirror_symmetry(O):
    rng = np.random.default_rng(3)
    for y in rng.integers(0, 2 ** 32, 20000, dtype=np.uint64):
        y = int(y)
        assert O.normal_from_u32(2 ** 32 - 1 - y) == -O.normal_from_u32(y)
    assert abs(O.normal_from_u32(2 ** 32 - 1)) <= 6.33795775455378925 + 1e-15


def test_lr_normals_moments(O):
    z = O.lr_normals(0, 16, 0, 20000)
    assert abs(z.mean()) < 4 / np.sqrt(z.size)
    assert abs(z.var() - 1) < 5 * np.sqrt(2 / z.size)
    # distinct replicates and distinct dimensions are different streams
    z2 = O.lr_normals(1, 16, 0, 100)
    assert not np.allclose(z[:100], z2)
    assert abs(np.corrcoef(z[:, 0], z[:, 1])[0, 1]) < 0.05
