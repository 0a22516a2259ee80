"""CPU-side checks of the boundary: the C-ABI library loads and exports every entry point
include/qb.h declares (no compute calls without a GPU), and the binding fails loudly."""
import ctypes
import os
import re

import pytest

import paper_1503_07157_b200 as qbp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "qb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:qb_status|void|const char\s*\*|int64_t)\s+(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("qb_create", "qb_factor", "qb_destroy", "qb_stats", "qb_omega", "qb_orth", "rqb_svd",
                     "qb_status_string", "qb_last_error", "qb_create_dist", "qb_nccl_unique_id"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_1503_07157_b200 import build
    build.build()
    L = ctypes.CDLL(qbp.LIB_PATH)
    for name in declared_functions():
        assert hasattr(L, name), name


def test_status_strings():
    for s, name in [(0, "QB_OK"), (1, "QB_NOT_CONVERGED"), (2, "QB_ERR_INVALID_ARG"), (6, "QB_ERR_ORTH_BREAKDOWN")]:
        assert qbp.qb_status_string(s) == name


def test_null_arguments_rejected_without_gpu():
    L = qbp.lib()
    assert L.qb_create(None, 0, 0, None) == qbp.QB_ERR_INVALID_ARG
    assert L.qb_stats(None, None, 0, None) == qbp.QB_ERR_INVALID_ARG


def test_binding_has_no_cpu_fallback(monkeypatch, tmp_path):
    monkeypatch.setattr(qbp, "_lib", None)
    monkeypatch.setattr(qbp, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        qbp.lib()


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_1503_07157_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
