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


def test_reference_shim_compiles_links_and_maps_errors(tmp_path):
    """include/fnlh_b200_shim.hpp against the reference's own headers:
    a C++ unit using the reference's BlockSparsityPattern / Bsr / BlockVec compiles, links
    libfnlh_b200.so (and the reference's compiled sources, oracle/_ref), and a C ABI
    status comes back as the reference's exception taxonomy (without a GPU: the device
    error of fnlh_pattern_create; with one: a ShapeError for a mismatched shift)."""
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = "/root/reference/proj/src"
    ref = os.path.join(root, "oracle", "_ref", "libfnlh_ref.so")
    lib = os.path.join(root, "paper_2404_01407_b200", "libfnlh_b200.so")
    if not (os.path.isdir(src) and os.path.exists(ref) and os.path.exists(lib) and shutil.which("g++")):
        pytest.skip("needs the reference sources, oracle/_ref and the built library")
    prog = tmp_path / "shim.cpp"
    prog.write_text(r'''
#include <cstdio>
#include "fnlh_b200_shim.hpp"
int main() {
    using namespace fnlh;
    auto pat = std::make_shared<BlockSparsityPattern>();
    pat->b = 1; pat->rows = 2;
    pat->row_ptr = {0, 2, 4}; pat->col_idx = {0, 1, 0, 1}; pat->diag_idx = {0, 3}; pat->partition = {0, 0};
    try {
        PatternB200 p(*pat);
        Bsr<real> A5(pat);
        BlockVec<cplx> rhs(1, 2), x;
        std::vector<real> shift(3, 1.0);  // wrong size on purpose
        smoothed_solve_b200(p, A5, std::span<const real>(shift), 0.1, 2, rhs, x);
    } catch (const ShapeError& e) {
        std::printf("ShapeError: %s\n", e.what());
        return 0;
    } catch (const std::runtime_error& e) {
        std::printf("runtime_error: %s\n", e.what());
        return 0;
    }
    return 1;
}
''')
    exe = tmp_path / "shim"
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"), "-I", src, str(prog), "-o", str(exe),
           lib, ref, f"-Wl,-rpath,{os.path.dirname(lib)}:{os.path.dirname(ref)}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, (r.stdout, r.stderr)
    assert r.stdout.startswith(("ShapeError", "runtime_error: fnlh_b200")), r.stdout
