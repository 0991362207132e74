"""ctypes binding of the plain-C QMC-CPW oracle (oracle/qmccpw_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
package paper_2209_11337_b200 never imports it (tests/test_independence.py
checks that), and it imports nothing from the product package.
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "qmccpw_oracle.c")
LIB = os.path.join(HERE, "libqmccpw_oracle.so")
JOE_KUO = os.path.join(HERE, "data", "new-joe-kuo-6.1024.txt")

ARITH, BINARY, LOOKBACK, GEOM_CALL, GEOM_DIGITAL = 0, 1, 2, 100, 101
STD, BB, PCA, GPCA = 0, 1, 2, 3
W1, X1 = 0, 1
QMC_CPW, LR_MC, MC_CPW, MC_AV_CPW = 0, 1, 2, 3
RAND_LMS_SHIFT, RAND_SHIFT, RAND_NONE, RAND_OWEN = 0, 1, 3, 4
DEFAULT_SEED = 2209113370


class Market(ctypes.Structure):
    _fields_ = [("S0", ctypes.c_double), ("r", ctypes.c_double), ("sigma", ctypes.c_double),
                ("T", ctypes.c_double), ("d", ctypes.c_int32)]


class Option(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int32), ("K", ctypes.c_double)]


class Config(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("construction", ctypes.c_int32),
                ("conditioning", ctypes.c_int32), ("randomization", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("point_offset", ctypes.c_uint64)]


class Result(ctypes.Structure):
    _fields_ = [("mean", ctypes.c_double * 4), ("se", ctypes.c_double * 4),
                ("sigma_run", ctypes.c_double * 4), ("within_var", ctypes.c_double * 4),
                ("n_points", ctypes.c_uint64), ("n_replicates", ctypes.c_uint32),
                ("argmax_near_ties", ctypes.c_uint64), ("mean_abs", ctypes.c_double * 4)]


def build(force=False):
    """Compile the oracle (plain gcc -O2, no -ffast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-o", LIB, SRC,
                               "-lm", "-lpthread"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P = ctypes.POINTER
        u32p, f64p = P(ctypes.c_uint32), P(ctypes.c_double)
        L.or_load_joe_kuo.argtypes = [ctypes.c_char_p]
        L.or_direction_numbers.argtypes = [ctypes.c_int32, u32p]
        L.or_polynomial.argtypes = [ctypes.c_int32, P(ctypes.c_int32), P(ctypes.c_int32)]
        L.or_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.or_philox4x32_10.restype = None
        L.or_randomization.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int32, u32p, u32p]
        L.or_sobol_u32.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                   ctypes.c_uint64, P(Config), u32p]
        L.or_sobol_from_vectors.argtypes = [u32p, u32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                            ctypes.c_uint64, u32p]
        L.or_owen_scramble.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.or_owen_scramble.restype = ctypes.c_uint32
        L.or_inv_normal_cdf.argtypes = [ctypes.c_double]
        L.or_inv_normal_cdf.restype = ctypes.c_double
        L.or_normal_from_u32.argtypes = [ctypes.c_uint32]
        L.or_normal_from_u32.restype = ctypes.c_double
        L.or_normals.argtypes = [ctypes.c_uint32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64, P(Config), f64p]
        L.or_lr_normals.argtypes = [ctypes.c_uint32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_uint64, f64p]
        L.or_path_matrix.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, f64p]
        L.or_construct.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, f64p, f64p]
        L.or_path_matrix_gpca.argtypes = [P(Market), f64p]
        L.or_estimate.argtypes = [P(Option), P(Market), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, f64p, f64p]
        L.or_path_values.argtypes = [P(Option), P(Market), P(Config), ctypes.c_uint32, ctypes.c_uint64,
                                     ctypes.c_uint64, f64p]
        L.or_pivots.argtypes = [P(Option), P(Market), f64p]
        L.or_price_greeks.argtypes = [P(Option), ctypes.c_int32, P(Market), ctypes.c_uint64, ctypes.c_uint32,
                                      P(Config), ctypes.c_int32, P(Result), f64p]
        L.or_summarize.argtypes = [f64p, ctypes.c_int32, f64p, f64p, f64p]
        L.or_last_error.restype = ctypes.c_char_p
        n = L.or_load_joe_kuo(JOE_KUO.encode())
        if n < 1024:
            raise RuntimeError(f"oracle: Joe-Kuo table load failed ({n})")
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().or_last_error().decode())


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _u32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _f64(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def config(method=QMC_CPW, construction=STD, conditioning=W1, randomization=RAND_LMS_SHIFT,
           seed=DEFAULT_SEED, point_offset=0):
    return Config(method, construction, conditioning, randomization, seed, point_offset)


def market(S0=100.0, r=0.1, sigma=0.2, T=1.0, d=64):
    return Market(S0, r, sigma, T, d)


# ---- thin wrappers -------------------------------------------------------
def direction_numbers(d):
    v = np.zeros((d, 32), np.uint32)
    _check(lib().or_direction_numbers(d, _u32(v)))
    return v


def polynomial(j):
    s, a = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().or_polynomial(j, ctypes.byref(s), ctypes.byref(a)))
    return s.value, a.value


def philox(ctr, key):
    c = np.asarray(ctr, np.uint32).copy()
    k = np.asarray(key, np.uint32).copy()
    out = np.zeros(4, np.uint32)
    lib().or_philox4x32_10(_u32(c), _u32(k), _u32(out))
    return out


def randomization(seed, rep, d, mode=RAND_LMS_SHIFT):
    v = np.zeros((d, 32), np.uint32)
    c = np.zeros(d, np.uint32)
    _check(lib().or_randomization(seed, rep, d, mode, _u32(v), _u32(c)))
    return v, c


def owen_scramble(y, seed):
    return int(lib().or_owen_scramble(int(y) & 0xFFFFFFFF, int(seed) & 0xFFFFFFFF))


def sobol_u32(rep, dim_begin, dim_end, k_begin, k_end, cfg=None):
    cfg = cfg or config()
    out = np.zeros((dim_end - dim_begin, k_end - k_begin), np.uint32)
    _check(lib().or_sobol_u32(rep, dim_begin, dim_end, k_begin, k_end, ctypes.byref(cfg), _u32(out)))
    return out


def sobol_from_vectors(v, shift, dim_begin, dim_end, k_begin, k_end):
    v = np.ascontiguousarray(v, np.uint32)
    shift = np.ascontiguousarray(shift, np.uint32)
    out = np.zeros((dim_end - dim_begin, k_end - k_begin), np.uint32)
    _check(lib().or_sobol_from_vectors(_u32(v), _u32(shift), dim_begin, dim_end, k_begin, k_end, _u32(out)))
    return out


def inv_normal_cdf(u):
    return lib().or_inv_normal_cdf(float(u))


def normal_from_u32(y):
    return lib().or_normal_from_u32(int(y))


def normals(rep, d, k_begin, k_end, cfg=None):
    cfg = cfg or config()
    out = np.zeros((k_end - k_begin, d))
    _check(lib().or_normals(rep, d, k_begin, k_end, ctypes.byref(cfg), _f64(out)))
    return out


def lr_normals(rep, d, k_begin, k_end, seed=DEFAULT_SEED):
    out = np.zeros((k_end - k_begin, d))
    _check(lib().or_lr_normals(rep, d, k_begin, k_end, seed, _f64(out)))
    return out


def path_matrix(construction, d, T=1.0):
    M = np.zeros((d, d))
    _check(lib().or_path_matrix(construction, d, T, _f64(M)))
    return M


def path_matrix_gpca(mk):
    M = np.zeros((mk.d, mk.d))
    _check(lib().or_path_matrix_gpca(ctypes.byref(mk), _f64(M)))
    return M


def construct(construction, x, T=1.0):
    x = np.ascontiguousarray(x, np.float64)
    W = np.zeros_like(x)
    _check(lib().or_construct(construction, len(x), T, _f64(x), _f64(W)))
    return W


def estimate(otype, K, mk, x, method=QMC_CPW, construction=STD, conditioning=W1):
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(4)
    opt = Option(otype, K)
    _check(lib().or_estimate(ctypes.byref(opt), ctypes.byref(mk), method, construction, conditioning,
                             _f64(x), _f64(out)))
    return out


def path_values(otype, K, mk, cfg, rep, k_begin, k_end):
    out = np.zeros((k_end - k_begin, 4))
    opt = Option(otype, K)
    _check(lib().or_path_values(ctypes.byref(opt), ctypes.byref(mk), ctypes.byref(cfg), rep, k_begin, k_end,
                                _f64(out)))
    return out


def pivots(otype, K, mk):
    out = np.zeros(4)
    opt = Option(otype, K)
    _check(lib().or_pivots(ctypes.byref(opt), ctypes.byref(mk), _f64(out)))
    return out


def summarize(C_l):
    c = np.ascontiguousarray(C_l, np.float64)
    m, se, sg = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _check(lib().or_summarize(_f64(c), len(c), ctypes.byref(m), ctypes.byref(se), ctypes.byref(sg)))
    return m.value, se.value, sg.value


def price_greeks(options, mk, n_points, n_replicates, cfg=None, n_threads=None, want_rep_means=False):
    """options: list of (type, K). Returns (list of dict results, rep_means[L, n_opt, 4] or None)."""
    cfg = cfg or config()
    n_threads = n_threads or os.cpu_count() or 1
    n_opt = len(options)
    opts = (Option * n_opt)(*[Option(t, K) for t, K in options])
    res = (Result * n_opt)()
    rm = np.zeros((n_replicates, n_opt, 4)) if want_rep_means else None
    _check(lib().or_price_greeks(opts, n_opt, ctypes.byref(mk), n_points, n_replicates, ctypes.byref(cfg),
                                 n_threads, res, _f64(rm) if rm is not None else None))
    out = []
    for r in res:
        out.append(dict(mean=np.array(r.mean[:]), se=np.array(r.se[:]), sigma_run=np.array(r.sigma_run[:]),
                        within_var=np.array(r.within_var[:]), n_points=r.n_points,
                        n_replicates=r.n_replicates, argmax_near_ties=r.argmax_near_ties,
                        mean_abs=np.array(r.mean_abs[:])))
    return out, rm
