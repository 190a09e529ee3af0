"""The drop-in at the reference's call sites: a reference-typed C++ unit
(tests/native/shim_stage_solve.cpp, built by oracle/Makefile against the reference's own
headers and compiled sources) runs the harmonic worker's factorize-once / solve-per-stage
sequence (driver.cpp:213-216, rk.cpp:82-85) through include/fnlh_b200_shim.hpp's persistent
handles and through the reference itself, on 2-colour and general patterns: iterates
bitwise equal, equal iteration counts, device bytes carried by the reference's LHS
accounting (sparse.hpp:34-37), and a stage solve launching only sweep kernels."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "shim_stage_solve")

pytestmark = pytest.mark.gpu


def test_shim_stage_solves_bitwise_against_reference():
    if not os.path.exists(EXE):
        pytest.fail("oracle/_ref/shim_stage_solve missing: build() compiles it where the reference sources exist")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
