"""Build libqmccpw.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

The kernels are split over several translation units (path kernels W1 / X1, PCA
W1 / X1, portfolio, tables + hooks, the C ABI, the roof microbenchmark) that are
compiled in parallel and linked into one shared library."""
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SOURCES = [os.path.join(CSRC, f) for f in (
    "qmccpw_paths_w1.cu", "qmccpw_paths_x1.cu", "qmccpw_pca_w1.cu", "qmccpw_pca_x1.cu", "qmccpw_pca_x1_owen.cu", "qmccpw_pca_x1_lb.cu",
    "qmccpw_portfolio.cu",
    "qmccpw_kernels.cu", "qmccpw_api.cu", "qmccpw_microbench.cu")]
HEADERS = [os.path.join(CSRC, f) for f in (
    "qmccpw_internal.h", "qmccpw_math.cuh", "qmccpw_coeffs.cuh", "qmccpw_device.cuh", "qmccpw_paths.cuh",
    "qmccpw_pca.cuh")] + [os.path.join(ROOT, "include", "qmccpw.h")]
LIB = os.path.join(PKG, "libqmccpw.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-c"]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force=False, verbose=False, defines=(), out=None):
    """defines/out: build an experimental variant (e.g. -DQMCCPW_BB_MINB=7) to another
    file, selected at load time with QMCCPW_LIB=<path> (A/B timing in one GPU session)."""
    if out is None and not force and not stale():
        return LIB
    target = out or LIB
    # object files outside the repo: they are large and must not travel to the GPU box
    objdir = os.path.join(os.environ.get("QMCCPW_OBJDIR", "/tmp/qmccpw_obj"), os.path.basename(target) + ".o.d")
    os.makedirs(objdir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC] + CFLAGS + [f"-D{d}" for d in defines] + ["-o", obj, src]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    logs, objs, failed = [], [], []
    for src, obj, p in procs:
        so, se = p.communicate()
        logs.append(f"==== {os.path.basename(src)}\n{so}{se}")
        objs.append(obj)
        if p.returncode != 0:
            failed.append(src)
    info = os.path.join(PKG, "ptxas_info.txt" if out is None else os.path.basename(out) + ".ptxas.txt")
    with open(info, "w") as f:
        f.write("\n".join(logs))
    if failed:
        raise RuntimeError("nvcc failed for " + ", ".join(failed) + ":\n" + "\n".join(logs))
    res = subprocess.run([NVCC] + ARCH + ["-shared", "-o", target] + objs + ["-lcurand"], capture_output=True,
                         text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n" + res.stdout + res.stderr)
    if verbose:
        print("\n".join(logs))
    return target


CHECKED_LIB = os.path.join(PKG, "libqmccpw_checked.so")


def build_checked(force=False):
    """The QMCCPW_CHECKED variant (device-side bounds asserts, tests/test_memory_safety.py),
    built next to the production library; rebuilt when a source is newer."""
    if not force and os.path.exists(CHECKED_LIB) and all(
            os.path.getmtime(f) <= os.path.getmtime(CHECKED_LIB) for f in SOURCES + HEADERS):
        return CHECKED_LIB
    return build(defines=("QMCCPW_CHECKED=1",), out=CHECKED_LIB)


if __name__ == "__main__":
    build(force=True, verbose=True)
