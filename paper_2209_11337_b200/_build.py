"""Build libqmccpw.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SOURCES = [os.path.join(CSRC, f) for f in ("qmccpw_kernels.cu", "qmccpw_api.cu", "qmccpw_microbench.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("qmccpw_internal.h", "qmccpw_math.cuh")] + \
    [os.path.join(ROOT, "include", "qmccpw.h")]
LIB = os.path.join(PKG, "libqmccpw.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force=False, verbose=False, defines=(), out=None):
    """defines/out: build an experimental variant (e.g. -DQMCCPW_ACC_SMEM=1) to another
    file, selected at load time with QMCCPW_LIB=<path> (A/B timing in one GPU session)."""
    if out is None and not force and not stale():
        return LIB
    cmd = [NVCC] + FLAGS + [f"-D{d}" for d in defines] + ["-o", out or LIB] + SOURCES + ["-lcurand"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    with open(os.path.join(PKG, "ptxas_info.txt" if out is None else os.path.basename(out) + ".ptxas.txt"), "w") as f:
        f.write(res.stderr)
    if verbose:
        print(res.stderr)
    return out or LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
