"""Seeded synthetic workloads of BASELINE.json (configs C1-C5).

Holds NO arithmetic of the method: only the inputs (market, strikes, sizes,
seed, construction/conditioning choices) shared by the CUDA path, the oracle,
the tests and bench.py.  Every input is a deterministic function of the seed
(the Sobol' randomisation and LR normals are drawn inside each implementation
from the same counter-based Philox stream).
"""
SEED = 2209113370
S0, R, SIGMA, T = 100.0, 0.1, 0.2, 1.0          # the paper's setting
STRIKES = (90.0, 100.0, 110.0)
ARITH, BINARY, LOOKBACK = 0, 1, 2
STD, BB, PCA = 0, 1, 2
W1, X1 = 0, 1

CONFIGS = {
    # name: (options, d, n_points, n_replicates, [(construction, conditioning), ...])
    "C1": dict(options=[ARITH], d=4, n_points=1 << 10, n_replicates=8,
               modes=[(STD, W1), (BB, W1), (PCA, X1)]),
    "C2": dict(options=[BINARY], d=16, n_points=1 << 14, n_replicates=16,
               modes=[(PCA, X1), (PCA, W1), (STD, W1)]),
    "C3": dict(options=[LOOKBACK], d=64, n_points=1 << 18, n_replicates=32,
               modes=[(BB, W1), (PCA, W1)]),
    "C4": dict(options=[ARITH, BINARY, LOOKBACK], d=64, n_points=1 << 20, n_replicates=64,
               modes=[(BB, W1)]),
}
HEADLINE = "C4"


def c5_portfolio():
    """C5: 1024 mixed options (SURVEY.md 8(d) generator): family f = i >> 7 with
    sigma_f = (0.1, 0.2, 0.3, 0.4)[f & 3], T_f = (0.5, 1.0)[f >> 2]; m = i & 127,
    type = m mod 3, K = 70 + 60 m / 127; d = 128."""
    out = []
    for i in range(1024):
        f, m = i >> 7, i & 127
        out.append(dict(type=m % 3, K=70.0 + 60.0 * m / 127.0, sigma=(0.1, 0.2, 0.3, 0.4)[f & 3],
                        T=(0.5, 1.0)[f >> 2], S0=S0, r=R, d=128))
    return out
