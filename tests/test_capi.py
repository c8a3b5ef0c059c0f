"""CPU: libgmds.so loads here (no GPU) and exports every symbol include/gmds.h declares."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gmds.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gmds_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "gmds_pairwise_gini" in syms and "gmds_minimize_stress" in syms and len(syms) > 20


def test_library_exports_every_declared_symbol():
    from paper_2605_25124_b200 import gmds

    L = gmds.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_no_device_fails_loudly():
    from paper_2605_25124_b200 import gmds

    if gmds.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(gmds.CudaError):
        gmds.pairwise_matrix([[0.0, 1.0], [2.0, 3.0]], 2.0)
    # argument validation happens first and mirrors the reference exception classes
    with pytest.raises(gmds.InvalidConfig):
        gmds.pairwise_matrix([[0.0, 1.0], [2.0, 3.0]], 1.0)
