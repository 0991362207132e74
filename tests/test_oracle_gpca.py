"""Pins of the oracle's GPCA path matrix, O5b (
DESIGN.md reading 28), each against something other than the oracle's own formula:

  * M M^T = C = [min(t_i, t_j)] (any valid construction must reproduce the covariance);
  * the first column equals C s / sqrt(s^T C s), s_j = exp(omega t_j), formed here
    from C and s directly;
  * M^T s is parallel to e_1 (the defining property: the linear part of the average
    loads on x_1 only);
  * M = M_pca Q with Q orthogonal (a rotation of the pinned PCA basis);
  * the per-path estimators under GPCA equal quadrature of the raw payoff (W1 and X1,
    all three options) and finite differences in S0 (M does not depend on S0);
  * GPCA estimates agree with the other constructions' within their standard errors.
"""
import math

import numpy as np
import pytest
from scipy import integrate, optimize

import oracle as O

S0, R, SIG, T = 100.0, 0.1, 0.2, 1.0


def cov(d, T):
    t = np.arange(1, d + 1) * T / d
    return np.minimum.outer(t, t), t


@pytest.mark.parametrize("d", [1, 2, 4, 16, 64, 128])
@pytest.mark.parametrize("r,sg,TT", [(0.1, 0.2, 1.0), (0.02, 0.5, 2.0), (-0.05, 0.3, 0.5)])
def test_gpca_is_a_rotation_aligned_with_the_average_gradient(d, r, sg, TT):
    M = O.path_matrix_gpca(O.market(S0, r, sg, TT, d))
    C, t = cov(d, TT)
    assert np.max(np.abs(M @ M.T - C)) <= 1e-13 * TT
    s = np.exp((r - 0.5 * sg * sg) * t)
    col = C @ s / math.sqrt(s @ C @ s)
    assert np.max(np.abs(M[:, 0] - col)) <= 1e-13 * math.sqrt(TT)
    assert np.all(M[:, 0] > 0) and np.all(np.diff(M[:, 0]) > 0)   # positive, increasing: X1's Newton and envelope
    g = M.T @ s
    assert np.all(np.abs(g[1:]) <= 1e-13 * abs(g[0]))
    P = O.path_matrix(O.PCA, d, TT)
    Q = np.linalg.solve(P, M)
    assert np.max(np.abs(Q.T @ Q - np.eye(d))) <= 1e-11


def raw(otype, K, S):
    D = math.exp(-R * T)
    if otype == 0:
        return D * max(S.mean() - K, 0.0)
    if otype == 1:
        return D * (1.0 if S.mean() > K else 0.0)
    return D * max(S.max() - K, 0.0)


def phi(u):
    return math.exp(-0.5 * u * u) / math.sqrt(2 * math.pi)


def quad(otype, K, S_of, kinks=()):
    stat = (lambda S: S.max()) if otype == 2 else (lambda S: S.mean())
    thr = optimize.brentq(lambda u: stat(S_of(u)) - K, -60, 60, xtol=1e-15, rtol=1e-15)
    f = lambda u: raw(otype, K, S_of(u)) * phi(u)
    pts = [thr] + sorted(k for k in kinks if thr < k < thr + 40) + [thr + 40]
    return sum(integrate.quad(f, a, b, epsabs=1e-15, epsrel=1e-13, limit=400)[0] for a, b in zip(pts[:-1], pts[1:]))


@pytest.mark.parametrize("otype", [0, 1, 2])
@pytest.mark.parametrize("cond", [0, 1])
def test_gpca_estimators_equal_quadrature_of_the_raw_payoff(otype, cond):
    rng = np.random.default_rng(31 + otype + 10 * cond)
    om = R - 0.5 * SIG * SIG
    for d in (4, 16):
        mk = O.market(S0, R, SIG, T, d)
        M = O.path_matrix_gpca(mk)
        t = np.arange(1, d + 1) * T / d
        for _ in range(3):
            x = rng.standard_normal(d)
            kinks = ()
            if cond:   # X1: condition on x_1
                Rj = M[:, 1:] @ x[1:]
                S_of = lambda u: S0 * np.exp(om * t + SIG * (Rj + M[:, 0] * u))
                if otype == 2:
                    c, b = om * t + SIG * Rj, SIG * M[:, 0]
                    kinks = [(c[i] - c[j]) / (b[j] - b[i]) for i in range(d) for j in range(i + 1, d)]
            else:      # W1: condition on W(t_1)
                W = M @ x
                Wt, t1 = W - W[0], t[0]
                S_of = lambda xi: S0 * np.exp(om * t + SIG * Wt + SIG * math.sqrt(t1) * xi)
            for K in (90.0, 100.0, 110.0):
                got = O.estimate(otype, K, mk, x, construction=O.GPCA, conditioning=cond)[0]
                ref = quad(otype, K, S_of, kinks)
                assert abs(got - ref) <= 1e-12 * max(1.0, abs(ref)), (d, K, got, ref)


@pytest.mark.parametrize("otype", [0, 1, 2])
@pytest.mark.parametrize("cond", [0, 1])
def test_gpca_delta_gamma_equal_finite_differences(otype, cond):
    rng = np.random.default_rng(5 + otype + 10 * cond)
    for d in (4, 64):
        x = 0.7 * rng.standard_normal(d)
        est = lambda s0: O.estimate(otype, 100.0, O.market(s0, R, SIG, T, d), x, construction=O.GPCA,
                                    conditioning=cond)
        g = est(S0)
        scale = np.abs(O.pivots(otype, 100.0, O.market(S0, R, SIG, T, d)))
        # steps inside the smoothing scale; the lookback under X1 has envelope kinks every
        # ~1/d of that scale, where G'' jumps and a wider stencil loses its accuracy
        h = (0.001 if (otype == 2 and cond) else 0.01) * S0 * SIG * math.sqrt(T / d)
        D = lambda f, hh: (f(S0 + hh) - f(S0 - hh)) / (2 * hh)
        fd = lambda f: (4 * D(f, h / 2) - D(f, h)) / 3
        assert abs(g[1] - fd(lambda s: est(s)[0])) <= 5e-8 * (abs(g[1]) + scale[1])
        assert abs(g[3] - fd(lambda s: est(s)[1])) <= 1e-7 * (abs(g[3]) + scale[3])


def test_gpca_agrees_with_the_other_constructions():
    d, N, L = 16, 1 << 12, 16
    mk = O.market(d=d)
    opts = [(0, 100.0), (1, 100.0), (2, 100.0)]
    ref, _ = O.price_greeks(opts, mk, N, L, O.config(construction=O.BB))
    for cond in (0, 1):
        got, _ = O.price_greeks(opts, mk, N, L, O.config(construction=O.GPCA, conditioning=cond))
        for o in range(3):
            for q in range(4):
                comb = math.hypot(got[o]["se"][q], ref[o]["se"][q])
                assert abs(got[o]["mean"][q] - ref[o]["mean"][q]) <= 4.5 * comb + 1e-12 * abs(ref[o]["mean"][q])
