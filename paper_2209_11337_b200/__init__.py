"""Python binding of libqmccpw.so, the B200-native QMC-CPW hot path.

Argument marshalling only: every step of the estimator runs in the sm_100a
kernels behind the C ABI declared in include/qmccpw.h (same function names).
There is no CPU fallback -- importing this package on a machine without the
built library raises, and every compute call without an sm_100a device
returns QMCCPW_ECUDA, surfaced here as QmcCpwError.
"""
import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QMCCPW_LIB") or os.path.join(_PKG, "libqmccpw.so")  # QMCCPW_LIB: A/B variants

OK, EINVAL, EUNSUPPORTED, ECUDA, ENOMEM = 0, -1, -2, -3, -4
ARITH_ASIAN_CALL, BINARY_ASIAN_CALL, LOOKBACK_CALL = 0, 1, 2
STD, BB, PCA, GPCA = 0, 1, 2, 3
COND_W1, COND_X1 = 0, 1
QMC_CPW, LR_MC, MC_CPW, MC_AV_CPW = 0, 1, 2, 3
RAND_LMS_SHIFT, RAND_SHIFT, RAND_CURAND_COMPAT, RAND_NONE, RAND_OWEN = 0, 1, 2, 3, 4
DEFAULT_SEED = 2209113370
CELL_POINTS = 4096
OUTPUTS = ("price", "delta", "vega", "gamma")


class QmcCpwError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"qmccpw error {code}: {msg}")
        self.code = code


class Params(ctypes.Structure):
    _fields_ = [("S0", ctypes.c_double), ("K", ctypes.c_double), ("r", ctypes.c_double),
                ("sigma", ctypes.c_double), ("T", ctypes.c_double), ("d", ctypes.c_int32)]


class Config(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("construction", ctypes.c_int32),
                ("conditioning", ctypes.c_int32), ("randomization", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("point_offset", ctypes.c_uint64),
                ("device", ctypes.c_int32), ("stream", ctypes.c_void_p)]


class Result(ctypes.Structure):
    _fields_ = [("mean", ctypes.c_double * 4), ("se", ctypes.c_double * 4),
                ("sigma_run", ctypes.c_double * 4), ("within_var", ctypes.c_double * 4),
                ("n_points", ctypes.c_uint64), ("n_replicates", ctypes.c_uint32),
                ("newton_unconverged", ctypes.c_uint64), ("argmax_near_ties", ctypes.c_uint64)]

    def as_dict(self):
        return dict(mean=np.array(self.mean[:]), se=np.array(self.se[:]), sigma_run=np.array(self.sigma_run[:]),
                    within_var=np.array(self.within_var[:]), n_points=self.n_points,
                    n_replicates=self.n_replicates, newton_unconverged=self.newton_unconverged,
                    argmax_near_ties=self.argmax_near_ties)


def params(S0=100.0, K=100.0, r=0.1, sigma=0.2, T=1.0, d=64):
    return Params(S0, K, r, sigma, T, d)


def config(method=QMC_CPW, construction=BB, conditioning=COND_W1, randomization=RAND_LMS_SHIFT,
           seed=DEFAULT_SEED, point_offset=0, device=-1, stream=None):
    return Config(method, construction, conditioning, randomization, seed, point_offset, device, stream)


_lib = None


def lib():
    """Load libqmccpw.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python __graft_entry__.py build` "
                              "(nvcc, sm_100a); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        u32p, f64p, u64p = P(ctypes.c_uint32), P(ctypes.c_double), P(ctypes.c_uint64)
        L.qmccpw_price_greeks.argtypes = [ctypes.c_int32, P(Params), ctypes.c_uint64, ctypes.c_uint32,
                                          P(Config), P(Result)]
        L.qmccpw_price_greeks_batch.argtypes = [P(ctypes.c_int32), P(Params), ctypes.c_int32, ctypes.c_uint64,
                                                ctypes.c_uint32, P(Config), P(Result)]
        L.qmccpw_cell_count.argtypes = [P(Params), ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint32, P(Config),
                                        u64p, u64p]
        L.qmccpw_partials.argtypes = [P(ctypes.c_int32), P(Params), ctypes.c_int32, ctypes.c_uint64,
                                      ctypes.c_uint32, P(Config), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
        L.qmccpw_replicate_sums.argtypes = [ctypes.c_void_p, P(Params), ctypes.c_int32, ctypes.c_uint64,
                                            ctypes.c_uint32, P(Config), ctypes.c_uint32, ctypes.c_uint32,
                                            ctypes.c_void_p]
        L.qmccpw_finalize.argtypes = [f64p, P(ctypes.c_int32), P(Params), ctypes.c_int32, ctypes.c_uint64,
                                      ctypes.c_uint32, P(Config), P(Result)]
        L.qmccpw_finalize_device.argtypes = [ctypes.c_void_p, P(ctypes.c_int32), P(Params), ctypes.c_int32,
                                             ctypes.c_uint64, ctypes.c_uint32, P(Config), P(Result)]
        L.qmccpw_sobol_u32.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                       ctypes.c_uint64, P(Config), u32p]
        L.qmccpw_normals.argtypes = [ctypes.c_uint32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64, P(Config),
                                     f64p]
        L.qmccpw_path_values.argtypes = [ctypes.c_int32, P(Params), ctypes.c_uint32, ctypes.c_uint64,
                                         ctypes.c_uint64, P(Config), f64p]
        L.qmccpw_portfolio_path_values.argtypes = [P(ctypes.c_int32), P(Params), ctypes.c_int32, ctypes.c_uint32,
                                                   ctypes.c_uint64, ctypes.c_uint64, P(Config), f64p]
        L.qmccpw_fp64_roof.argtypes = [ctypes.c_int32, f64p, f64p, f64p, f64p]
        L.qmccpw_last_error.restype = ctypes.c_char_p
        L.qmccpw_release.argtypes = [ctypes.c_int32]
        L.qmccpw_release.restype = None
        L.qmccpw_launch_count.argtypes = [ctypes.c_int32]
        L.qmccpw_launch_count.restype = ctypes.c_uint64
        _lib = L
    return _lib


def _check(rc):
    if rc != OK:
        raise QmcCpwError(rc, lib().qmccpw_last_error().decode())


def _cfg(cfg):
    return ctypes.byref(cfg) if cfg is not None else None


def qmccpw_price_greeks(option, p, n_points, n_replicates, cfg=None):
    out = Result()
    _check(lib().qmccpw_price_greeks(option, ctypes.byref(p), n_points, n_replicates, _cfg(cfg), ctypes.byref(out)))
    return out


def qmccpw_price_greeks_batch(options, plist, n_points, n_replicates, cfg=None):
    n = len(options)
    opts = (ctypes.c_int32 * n)(*options)
    ps = (Params * n)(*plist)
    out = (Result * n)()
    _check(lib().qmccpw_price_greeks_batch(opts, ps, n, n_points, n_replicates, _cfg(cfg), out))
    return list(out)


def qmccpw_cell_count(p, n_options, n_points, n_replicates, cfg=None):
    nc, pd = ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib().qmccpw_cell_count(ctypes.byref(p), n_options, n_points, n_replicates, _cfg(cfg),
                                   ctypes.byref(nc), ctypes.byref(pd)))
    return nc.value, pd.value


def qmccpw_partials(options, plist, n_points, n_replicates, cfg, cell_begin, cell_end, d_partials_ptr):
    n = len(options)
    _check(lib().qmccpw_partials((ctypes.c_int32 * n)(*options), (Params * n)(*plist), n, n_points, n_replicates,
                                 _cfg(cfg), cell_begin, cell_end, ctypes.c_void_p(d_partials_ptr)))


def qmccpw_replicate_sums(d_partials_ptr, p, n_options, n_points, n_replicates, cfg, rep_begin, rep_end,
                          d_rep_sums_ptr):
    _check(lib().qmccpw_replicate_sums(ctypes.c_void_p(d_partials_ptr), ctypes.byref(p), n_options, n_points,
                                       n_replicates, _cfg(cfg), rep_begin, rep_end, ctypes.c_void_p(d_rep_sums_ptr)))


def qmccpw_finalize(h_rep_sums, options, plist, n_points, n_replicates, cfg=None):
    n = len(options)
    rs = np.ascontiguousarray(h_rep_sums, np.float64)
    out = (Result * n)()
    _check(lib().qmccpw_finalize(rs.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), (ctypes.c_int32 * n)(*options),
                                 (Params * n)(*plist), n, n_points, n_replicates, _cfg(cfg), out))
    return list(out)


def qmccpw_finalize_device(d_partials_ptr, options, plist, n_points, n_replicates, cfg=None):
    n = len(options)
    out = (Result * n)()
    _check(lib().qmccpw_finalize_device(ctypes.c_void_p(d_partials_ptr), (ctypes.c_int32 * n)(*options),
                                        (Params * n)(*plist), n, n_points, n_replicates, _cfg(cfg), out))
    return list(out)


def qmccpw_sobol_u32(replicate, dim_begin, dim_end, k_begin, k_end, cfg=None):
    out = np.zeros((dim_end - dim_begin, k_end - k_begin), np.uint32)
    _check(lib().qmccpw_sobol_u32(replicate, dim_begin, dim_end, k_begin, k_end, _cfg(cfg),
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
    return out


def qmccpw_normals(replicate, d, k_begin, k_end, cfg=None):
    out = np.zeros((k_end - k_begin, d))
    _check(lib().qmccpw_normals(replicate, d, k_begin, k_end, _cfg(cfg),
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return out


def qmccpw_path_values(option, p, replicate, k_begin, k_end, cfg=None):
    out = np.zeros((k_end - k_begin, 4))
    _check(lib().qmccpw_path_values(option, ctypes.byref(p), replicate, k_begin, k_end, _cfg(cfg),
                                    out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return out


def qmccpw_fp64_roof(device=0):
    vals = [ctypes.c_double() for _ in range(4)]
    _check(lib().qmccpw_fp64_roof(device, *[ctypes.byref(v) for v in vals]))
    return dict(dfma_tflops=vals[0].value, dfma_latency_cycles=vals[1].value, dmma_tflops=vals[2].value,
                sm_clock_mhz=vals[3].value)


def qmccpw_portfolio_path_values(options, plist, replicate, k_begin, k_end, cfg=None):
    n = len(options)
    out = np.zeros((k_end - k_begin, n, 4))
    _check(lib().qmccpw_portfolio_path_values((ctypes.c_int32 * n)(*options), (Params * n)(*plist), n, replicate,
                                              k_begin, k_end, _cfg(cfg),
                                              out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return out


def qmccpw_last_error():
    return lib().qmccpw_last_error().decode()


def qmccpw_release(device=-1):
    lib().qmccpw_release(device)


def qmccpw_launch_count(reset=False):
    return lib().qmccpw_launch_count(1 if reset else 0)
