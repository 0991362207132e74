"""Pins for oracle step O5 (path constructions W = M x).

External references: the Brownian covariance C_ij = min(t_i, t_j) that every
construction must reproduce, SPEC.md's hand traces of
Alg. 4 at d = 2, a hand trace of Alg. 4 at d = 4 (below),
the terminal identity of the bridge, and LAPACK's eigh for PCA.
"""
import numpy as np
import pytest


def cov(d, T):
    t = np.arange(1, d + 1) * T / d
    return np.minimum.outer(t, t)


@pytest.mark.parametrize("constr,d", [(0, 1), (0, 5), (0, 64), (1, 1), (1, 2), (1, 4), (1, 64), (1, 256),
                                      (2, 1), (2, 3), (2, 64), (2, 256)])
@pytest.mark.parametrize("T", [1.0, 0.5])
def test_MMt_is_brownian_covariance(O, constr, d, T):
    M = O.path_matrix(constr, d, T)
    assert np.max(np.abs(M @ M.T - cov(d, T))) <= 2e-14 * T


def test_std_is_cumulative_sum(O):
    x = np.array([0.3, -0.2, 0.5, 1.1])
    assert np.allclose(O.construct(0, x, 1.0), np.cumsum(0.5 * x), atol=1e-16)


def test_bb_spec_traces(O):
    # d = 2, T = 1: (1,0) -> increments (0.5, 0.5); (0,1) -> (0.5, -0.5)
    W = O.construct(1, np.array([1.0, 0.0]))
    assert np.allclose(np.diff(np.r_[0, W]), [0.5, 0.5], atol=0)
    W = O.construct(1, np.array([0.0, 1.0]))
    assert np.allclose(np.diff(np.r_[0, W]), [0.5, -0.5], atol=0)


def test_bb_d4_hand_trace(O):
    # Alg. 4 by hand at d = 4, T = 1, b_1 = 1/2, b_2 = 1/(2 sqrt 2):
    # path[0] = z0; level 1: j=0: path[1] = z0/2 - z1/2, path[0] = z0/2 + z1/2;
    # level 2: j=1: path[3] = path[1]/2 - b z2, path[2] = path[1]/2 + b z2;
    #          j=0: path[1] = path[0]/2 - b z3, path[0] = path[0]/2 + b z3.
    rng = np.random.default_rng(0)
    b = 1 / (2 * np.sqrt(2))
    for _ in range(20):
        z = rng.standard_normal(4)
        inc = [z[0] / 4 + z[1] / 4 + b * z[3], z[0] / 4 + z[1] / 4 - b * z[3],
               z[0] / 4 - z[1] / 4 + b * z[2], z[0] / 4 - z[1] / 4 - b * z[2]]
        assert np.allclose(O.construct(1, z), np.cumsum(inc), atol=1e-15)


@pytest.mark.parametrize("d", [1, 2, 8, 64, 256])
def test_bb_terminal_identity(O, d):
    # W(t_d) = sqrt(T) z_1 (to rounding of the prefix sum)
    rng = np.random.default_rng(d)
    for T in (1.0, 2.0):
        z = rng.standard_normal(d)
        assert abs(O.construct(1, z, T)[-1] - np.sqrt(T) * z[0]) <= 1e-14 * (1 + abs(z[0]))


@pytest.mark.parametrize("d", [2, 4, 16, 64, 128])
def test_pca_is_the_eigendecomposition(O, d):
    T = 1.0
    M = O.path_matrix(2, d, T)
    lam = np.sum(M * M, axis=0)              # column norms^2 = eigenvalues
    ref = np.linalg.eigvalsh(cov(d, T))[::-1]
    assert np.max(np.abs(lam - ref)) <= 1e-13 * ref[0]
    assert np.all(np.diff(lam) < 0)          # descending (reading 18)
    G = M.T @ M                               # orthogonal columns
    assert np.max(np.abs(G - np.diag(lam))) <= 1e-14 * ref[0]
    assert np.all(M[:, 0] > 0)                # first column positive (needed by X1 mode)
    # scaling M(T) = sqrt(T) M(1)
    assert np.allclose(O.path_matrix(2, d, 0.25), 0.5 * M, rtol=1e-14, atol=0)
