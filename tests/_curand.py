"""ctypes access to NVIDIA's libcurand HOST API (runs on the CPU, no GPU needed).

The paper generates its points with cuRAND's QUASI_SCRAMBLED_SOBOL32 and
PSEUDO generators.  libcurand is an external implementation of
the same definitions, so it pins the oracle's direction numbers, Gray-code
ordering, digital shift and Philox bit-exactly.  Test helper only.
"""
import ctypes
import os

import numpy as np

PATH = "/usr/local/cuda/lib64/libcurand.so"
QUASI_SOBOL32 = 201
QUASI_SCRAMBLED_SOBOL32 = 202
PSEUDO_PHILOX4_32_10 = 161
DIRECTION_VECTORS_32_JOEKUO6 = 101
SCRAMBLED_DIRECTION_VECTORS_32_JOEKUO6 = 102


def available():
    return os.path.exists(PATH)


def _lib():
    return ctypes.CDLL(PATH)


def direction_vectors(scrambled=False, ndim=1024):
    L = _lib()
    ptr = ctypes.POINTER(ctypes.c_uint32)()
    rc = L.curandGetDirectionVectors32(ctypes.byref(ptr), SCRAMBLED_DIRECTION_VECTORS_32_JOEKUO6 if scrambled
                                       else DIRECTION_VECTORS_32_JOEKUO6)
    assert rc == 0
    return np.ctypeslib.as_array(ptr, shape=(20000 * 32,)).reshape(20000, 32)[:ndim].copy()


def scramble_constants(ndim=1024):
    L = _lib()
    ptr = ctypes.POINTER(ctypes.c_uint32)()
    assert L.curandGetScrambleConstants32(ctypes.byref(ptr)) == 0
    return np.ctypeslib.as_array(ptr, shape=(20000,))[:ndim].copy()


def host_generate(rng_type, n_per_dim, ndim=1, seed=None, offset=0):
    """Returns uint32 array [ndim][n_per_dim] (cuRAND quasi output is dimension-major)."""
    L = _lib()
    gen = ctypes.c_void_p()
    assert L.curandCreateGeneratorHost(ctypes.byref(gen), rng_type) == 0
    try:
        if rng_type in (QUASI_SOBOL32, QUASI_SCRAMBLED_SOBOL32):
            assert L.curandSetQuasiRandomGeneratorDimensions(gen, ctypes.c_uint(ndim)) == 0
        if seed is not None:
            assert L.curandSetPseudoRandomGeneratorSeed(gen, ctypes.c_ulonglong(seed)) == 0
        if offset:
            assert L.curandSetGeneratorOffset(gen, ctypes.c_ulonglong(offset)) == 0
        out = np.zeros(ndim * n_per_dim, np.uint32)
        rc = L.curandGenerate(gen, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), ctypes.c_size_t(out.size))
        assert rc == 0, rc
    finally:
        L.curandDestroyGenerator(gen)
    return out.reshape(ndim, n_per_dim)
