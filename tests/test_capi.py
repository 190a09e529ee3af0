"""CPU: the C-ABI library loads without a GPU and exports every entry point that
include/fnlh_b200.h declares; the product refuses to run without a device (no
CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    txt = open(os.path.join(ROOT, "include", "fnlh_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fnlh_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    from paper_2404_01407_b200._lib import LIB_PATH
    lib = ctypes.CDLL(LIB_PATH)
    names = declared()
    assert len(names) > 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_no_cpu_fallback():
    from paper_2404_01407_b200._lib import lib, require_gpu
    if lib().fnlh_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError):
        require_gpu()
    from paper_2404_01407_b200 import la
    from paper_2404_01407_b200._lib import FnlhError
    with pytest.raises(FnlhError) as e:
        la.Pattern(1, [0, 1], [0])
    assert e.value.kind == "CudaError"


def test_error_taxonomy_matches_reference():
    from paper_2404_01407_b200._lib import STATUS
    assert STATUS == {1: "ConfigError", 2: "StateError", 3: "ShapeError", 4: "UnsupportedCaseError",
                      5: "FactorizationError", 6: "DivergenceError", 7: "CudaError", 8: "NonConvergenceError"}
