"""Regenerate oracle/data/new-joe-kuo-6.1024.txt (Joe-Kuo direction-number PARAMETERS).

TEST INFRASTRUCTURE ONLY (oracle data provenance).

The paper draws its Sobol' points from cuRAND's QUASI_SCRAMBLED_SOBOL32
generator (Sec. 4.1), whose direction numbers are the Joe-Kuo
"new-joe-kuo-6" set.  There is no network here, so the published parameter
file cannot be downloaded; instead this script reads cuRAND's *expanded*
32-bit direction vectors (curandGetDirectionVectors32, JOEKUO6) and recovers,
for every dimension 2..1024, the unique (s, a, m_1..m_s) such that the
recurrence of PAPER.md:166 (Sec. 2.2.2)

    m_k = 2 c_1 m_{k-1} ^ 4 c_2 m_{k-2} ^ ... ^ 2^{s-1} c_{s-1} m_{k-s+1}
          ^ 2^s m_{k-s} ^ m_{k-s},       c_i = bit (s-1-i) of a,

reproduces all 32 of cuRAND's numbers.  Only the PARAMETERS are written; the
oracle expands them with its own code (oracle/qmccpw_oracle.c, O1), and the
tests pin that expansion against cuRAND again and against the Joe-Kuo rows
quoted in SURVEY.md Appendix B6.  Dimension 1 is the van der Corput identity
 and is not listed, as in the Joe-Kuo file format.
"""
import ctypes
import os
import sys

import numpy as np

CURAND = "/usr/local/cuda/lib64/libcurand.so"
JOEKUO6 = 101
NDIM = 1024


def curand_vectors():
    lib = ctypes.CDLL(CURAND)
    ptr = ctypes.POINTER(ctypes.c_uint32)()
    rc = lib.curandGetDirectionVectors32(ctypes.byref(ptr), JOEKUO6)
    if rc != 0:
        raise RuntimeError(f"curandGetDirectionVectors32 failed: {rc}")
    return np.ctypeslib.as_array(ptr, shape=(20000 * 32,)).reshape(20000, 32).copy()


def expand(s, a, m_init):
    m = list(m_init)
    for k in range(s, 32):  # 0-based k -> m_{k+1}
        new = m[k - s] ^ (m[k - s] << s)
        for i in range(1, s):
            if (a >> (s - 1 - i)) & 1:
                new ^= m[k - i] << i
        m.append(new)
    return m


def fit(vec):
    m_all = [int(vec[b]) >> (31 - b) for b in range(32)]
    for s in range(1, 19):
        for a in range(1 << (s - 1)):
            if expand(s, a, m_all[:s]) == m_all:
                return s, a, m_all[:s]
    raise RuntimeError("no fit")


def main(out_path):
    v = curand_vectors()
    assert all(int(v[0][b]) == 1 << (31 - b) for b in range(32)), "dim 1 must be the identity"
    lines = ["d       s       a       m_i"]
    for dim in range(2, NDIM + 1):
        s, a, m = fit(v[dim - 1])
        lines.append(f"{dim}\t{s}\t{a}\t" + " ".join(str(x) for x in m))
    with open(out_path, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(f"wrote {out_path}: dims 2..{NDIM}")


if __name__ == "__main__":
    here = os.path.dirname(os.path.abspath(__file__))
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(here, "..", "data", "new-joe-kuo-6.1024.txt"))
