"""Memory-safety checks of the sm_100a kernels without compute-sanitizer.

compute-sanitizer is closed on the GPU pool (profiles/r02/sanitizer_closed_on_pool.log: every
tool exits 86), so its four tools are replaced by checks of our own:

  memcheck   -> the QMCCPW_CHECKED build (libqmccpw_checked.so): device-side bounds asserts at
                the computed shared- and global-memory indices (every Sobol' table read and
                write, the staging, the bridge stack, the hull, the X1 columns, the partial
                rows, the hook outputs); a violation traps and the call fails.  It runs the
                every-kernel call list and must agree with the production build;
  initcheck  -> QMCCPW_POISON=1 fills the library's scratch (tables, partials, replicate
                sums) with 0xFF bytes (NaN) on every call: results must be bit-identical, so no
                kernel reads scratch it did not write; caller-owned partial rows outside the
                launch's cells must keep a sentinel (no write outside its cells);
  racecheck /
  synccheck  -> bit-identical results over repeated launches and over two streams running
                concurrently on one device (a shared-memory race or a missing barrier shows
                up as run-to-run differences in the fixed-order reductions).
"""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tests", "tools", "safety_calls.py")


@pytest.fixture(scope="module")
def q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2209_11337_b200 as q
    q.lib()
    return q


def _run(env_extra, out):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, TOOL, out], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return np.load(out)


@pytest.fixture(scope="module")
def reference_values(q):
    with tempfile.TemporaryDirectory() as d:
        return _run({}, os.path.join(d, "ref.npy"))


def test_poisoned_scratch_gives_bit_identical_results(reference_values):
    with tempfile.TemporaryDirectory() as d:
        v = _run({"QMCCPW_POISON": "1"}, os.path.join(d, "poison.npy"))
    assert v.shape == reference_values.shape
    assert np.array_equal(v, reference_values, equal_nan=True)


def test_checked_build_traps_nothing_and_agrees(reference_values):
    from paper_2209_11337_b200 import _build
    lib = _build.build_checked()
    with tempfile.TemporaryDirectory() as d:
        v = _run({"QMCCPW_LIB": lib, "QMCCPW_POISON": "1"}, os.path.join(d, "checked.npy"))
    assert v.shape == reference_values.shape
    # the asserts change code generation (FMA contraction, scheduling) only around integer
    # index arithmetic: the FP64 results agree to rounding
    scale = np.maximum(np.abs(reference_values), 1e-300)
    assert np.all(np.abs(v - reference_values) <= 1e-12 * scale + 1e-300), np.max(np.abs(v - reference_values) / scale)


@pytest.mark.parametrize("constr,cond,opts,d", [(1, 0, [0, 1, 2], 64), (2, 0, [0, 1, 2], 64), (2, 1, [0, 1, 2], 64),
                                                (1, 1, [0, 1], 16), (2, 0, [0, 1, 2, 0, 1], 16)])
def test_partials_write_only_their_cells(q, constr, cond, opts, d):
    import torch
    N, L = 3 * 4096 + 5, 3
    cfg = q.config(construction=constr, conditioning=cond, device=0)
    ps = [q.params(K=90.0 + 5 * i, d=d) for i in range(len(opts))]
    n_cells, per = q.qmccpw_cell_count(ps[0], len(opts), N, L, cfg)
    sentinel = torch.full((n_cells * per,), float.fromhex("0x1.dead0beefp+600"), dtype=torch.float64, device="cuda:0")
    b, e = 2, n_cells - 3
    buf = sentinel.clone()
    buf[b * per:e * per] = 0.0
    q.qmccpw_partials(opts, ps, N, L, cfg, b, e, buf.data_ptr())
    torch.cuda.synchronize()
    h = buf.cpu().numpy().reshape(n_cells, per)
    s = sentinel[0].item()
    assert np.all(h[:b] == s) and np.all(h[e:] == s)          # nothing outside the launch's cells
    assert np.all(np.isfinite(h[b:e]))
    assert np.all(h[b:e, len(opts) * 8 + 2] > 0)              # every own cell evaluated its points
    # replicate sums write only [rep_begin, rep_end)
    rs = torch.full((L * per,), s, dtype=torch.float64, device="cuda:0")
    rs[per:2 * per] = 0.0
    q.qmccpw_replicate_sums(buf.data_ptr(), ps[0], len(opts), N, L, cfg, 1, 2, rs.data_ptr())
    torch.cuda.synchronize()
    r = rs.cpu().numpy().reshape(L, per)
    assert np.all(r[0] == s) and np.all(r[2] == s) and np.all(np.isfinite(r[1]))


def test_repeated_and_concurrent_launches_are_bit_identical(q):
    import torch
    N, L = 8 * 4096, 6
    opts = [0, 1, 2]
    modes = [(1, 0), (2, 0), (2, 1), (0, 1)]
    ps = [q.params(d=64)] * 3
    ref = {}
    for m in modes:
        runs = [q.qmccpw_price_greeks_batch(opts, ps, N, L, q.config(construction=m[0], conditioning=m[1], device=0))
                for _ in range(3)]
        arr = [np.array([r.mean[:] + r.se[:] for r in run]) for run in runs]
        assert all(np.array_equal(arr[0], a) for a in arr[1:]), m
        ref[m] = arr[0]
    # two modes on two streams at once: per-(device, stream) scratch keeps their tables apart
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    bufs = {}
    for m, s in zip(((1, 0), (2, 1)), (s1, s2)):
        cfg = q.config(construction=m[0], conditioning=m[1], device=0, stream=s.cuda_stream)
        n_cells, per = q.qmccpw_cell_count(ps[0], 3, N, L, cfg)
        bufs[m] = (torch.zeros(n_cells * per, dtype=torch.float64, device="cuda:0"), cfg)
    for _ in range(2):
        for m in bufs:
            bufs[m][0].zero_()
        torch.cuda.synchronize()
        for m in bufs:  # enqueue both without waiting: the kernels overlap on the device
            q.qmccpw_partials(opts, ps, N, L, bufs[m][1], 0, bufs[m][0].numel() // (3 * 8 + 3), bufs[m][0].data_ptr())
        torch.cuda.synchronize()
        for m in bufs:
            res = q.qmccpw_finalize_device(bufs[m][0].data_ptr(), opts, ps, N, L,
                                           q.config(construction=m[0], conditioning=m[1], device=0))
            assert np.array_equal(np.array([r.mean[:] + r.se[:] for r in res]), ref[m]), m
