"""CPU-side checks of the C ABI boundary: the library builds/loads, exports
every function include/qmccpw.h declares, validates arguments before touching
a device, and fails loudly (QMCCPW_ECUDA) instead of falling back when there
is no sm_100a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qmccpw.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qmccpw_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2209_11337_b200 as q
    q.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", q.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (qmccpw_\w+)", out))
    decl = declared_functions()
    assert len(decl) >= 11
    missing = [f for f in decl if f not in exported]
    assert not missing, missing


def test_library_is_sm100a_only():
    import paper_2209_11337_b200 as q
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", q.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(7|8|9)\d", out)


def test_validation_happens_before_device_access():
    import paper_2209_11337_b200 as q
    bad = [q.params(S0=-1.0), q.params(K=float("nan")), q.params(sigma=0.0), q.params(T=float("inf")),
           q.params(d=0), q.params(d=2000), q.params(r=float("nan"))]
    for p in bad:
        with pytest.raises(q.QmcCpwError) as e:
            q.qmccpw_price_greeks(0, p, 1024, 8, q.config(construction=q.STD))
        assert e.value.code == q.EINVAL
    with pytest.raises(q.QmcCpwError) as e:
        q.qmccpw_price_greeks(0, q.params(d=4), 0, 8, q.config(construction=q.STD))
    assert e.value.code == q.EINVAL
    with pytest.raises(q.QmcCpwError) as e:
        q.qmccpw_price_greeks(0, q.params(d=4), 1024, 0, q.config(construction=q.STD))
    assert e.value.code == q.EINVAL
    with pytest.raises(q.QmcCpwError) as e:
        q.qmccpw_price_greeks(0, q.params(d=4), 1 << 32, 1, q.config(construction=q.STD, point_offset=1))
    assert e.value.code == q.EINVAL
    for cfg, opt in ((q.config(construction=q.BB), 0),
                     (q.config(method=q.LR_MC, construction=q.PCA), 0),
                     (q.config(method=q.MC_CPW, construction=q.PCA), 0),
                     (q.config(method=q.MC_AV_CPW, construction=q.STD, conditioning=q.COND_X1), 0)):
        with pytest.raises(q.QmcCpwError) as e:
            q.qmccpw_price_greeks(opt, q.params(d=6), 1024, 8, cfg)
        assert e.value.code == q.EUNSUPPORTED
    with pytest.raises(q.QmcCpwError) as e:  # several (sigma, T) families need the PCA-W1 portfolio kernel
        q.qmccpw_price_greeks_batch([0, 1], [q.params(sigma=0.2, d=4), q.params(sigma=0.3, d=4)], 1024, 8,
                                    q.config(construction=q.STD))
    assert e.value.code == q.EUNSUPPORTED
    with pytest.raises(q.QmcCpwError) as e:  # more than 8 families
        q.qmccpw_price_greeks_batch([0] * 9, [q.params(sigma=0.1 + 0.01 * i, d=8) for i in range(9)], 1024, 2,
                                    q.config(construction=q.PCA))
    assert e.value.code == q.EUNSUPPORTED
    with pytest.raises(q.QmcCpwError) as e:  # GPCA (row f3) is one market per call, not a portfolio
        q.qmccpw_price_greeks_batch([0, 1, 2, 0], [q.params(K=90.0 + i, d=8) for i in range(4)], 1024, 2,
                                    q.config(construction=q.GPCA))
    assert e.value.code == q.EUNSUPPORTED
    for cfg in (q.config(construction=5), q.config(randomization=5), q.config(method=q.MC_CPW, construction=q.GPCA)):
        with pytest.raises(q.QmcCpwError) as e:
            q.qmccpw_price_greeks(0, q.params(d=8), 1024, 2, cfg)
        assert e.value.code in (q.EINVAL, q.EUNSUPPORTED)
    with pytest.raises(q.QmcCpwError) as e:  # different S0
        q.qmccpw_price_greeks_batch([0, 0], [q.params(S0=100.0, d=8), q.params(S0=90.0, d=8)], 1024, 2,
                                    q.config(construction=q.PCA))
    assert e.value.code == q.EUNSUPPORTED


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2209_11337_b200 as q
    with pytest.raises(q.QmcCpwError) as e:
        q.qmccpw_price_greeks(0, q.params(d=4), 1024, 8, q.config(construction=q.STD))
    assert e.value.code == q.ECUDA


def test_cell_count():
    import paper_2209_11337_b200 as q
    n, per = q.qmccpw_cell_count(q.params(d=64), 3, 1 << 20, 64, q.config())
    assert (n, per) == (64 * 256, 27)
    n, per = q.qmccpw_cell_count(q.params(d=4), 1, 4097, 3, q.config(construction=q.STD))
    assert (n, per) == (6, 11)
