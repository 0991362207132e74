"""The oracle and the CUDA path share no code: neither imports/includes the
other, and the product path never references oracle/ (task rule)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _files(d, exts):
    for dp, _, fs in os.walk(os.path.join(ROOT, d)):
        for f in fs:
            if f.endswith(exts):
                yield os.path.join(dp, f)


def test_product_never_references_oracle():
    for f in _files("paper_2209_11337_b200", (".py", ".cu", ".cuh", ".h", ".cpp")):
        src = open(f).read()
        assert not re.search(r"\bimport\s+oracle|from\s+oracle|qmccpw_oracle|\bor_[a-z_]+\(", src), f
    for f in _files("include", (".h",)):
        assert "oracle" not in open(f).read().lower().replace("independent of oracle", "")


def test_oracle_never_references_product():
    for f in _files("oracle", (".py", ".c", ".h")):
        src = open(f).read()
        assert "paper_2209_11337_b200" not in src.replace("paper_2209_11337_b200/", "") or f.endswith(".py") and \
            "import paper_2209_11337_b200" not in src, f
        assert "qmccpw.h" not in src and "qmccpw_internal" not in src, f


def test_workloads_module_has_no_method_arithmetic():
    src = open(os.path.join(ROOT, "workloads.py")).read()
    for token in ("exp(", "log(", "erfc", "sqrt", "import oracle", "paper_2209_11337_b200"):
        assert token not in src, token
