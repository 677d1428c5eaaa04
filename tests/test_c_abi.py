"""The C ABI library loads on CPU and exports every entry point include/gx.h declares."""
import os
import re

from paper_2211_13878_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gx.h")).read()
    return sorted(set(re.findall(r"GX_API\s+[\w\s\*]+?\b(gx_\w+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    L = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_oracle_ref_exports_same_plan_surface():
    from oracle import ref_planner
    if not ref_planner.available():
        import pytest
        pytest.skip("oracle/_ref not built")
    import ctypes
    R = ctypes.CDLL(ref_planner.REF_LIB)
    for n in declared_symbols():
        if n.startswith("gx_plan_"):
            assert hasattr(R, "ref_plan_" + n[len("gx_plan_"):]), n


def test_version_and_error_reporting():
    L = _lib.lib()
    assert L.gx_version() >= 1
    # a malformed strategy must fail with a validation error and a message, without CUDA
    import pytest
    from paper_2211_13878_b200 import planner
    with pytest.raises(_lib.ValidationError, match="unknown dimension"):
        planner.api().estimate(1, 1, 1.0, "xp:2", 8, 1.0)
