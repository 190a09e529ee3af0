"""Out-of-bounds checking without a sanitizer (compute-sanitizer is closed on this pool):
the guard build of the library (paper_2404_01407_b200/build.py build_guard: every device
buffer between 4 KiB guard zones of 0xFF bytes, the reference's CountedBuffer canaries,
sparse.hpp:40-100) runs two outer iterations of every solver path and the persistent
handles (profiles/guard_step.py).  No kernel may write into a guard zone, and every
residual must equal the product build's bit for bit (an out-of-bounds read would pull in
NaN guard bytes)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GUARD = os.path.join(ROOT, "paper_2404_01407_b200", "libfnlh_b200_guard.so")
pytestmark = pytest.mark.gpu


def _run(lib=None):
    env = dict(os.environ)
    if lib:
        env["FNLH_B200_LIB"] = lib
    r = subprocess.run([sys.executable, os.path.join(ROOT, "profiles", "guard_step.py")], capture_output=True,
                       text=True, timeout=1200, env=env, cwd=ROOT)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    return r.stdout.splitlines()


def test_guard_zones_intact_and_results_bitwise():
    if not os.path.exists(GUARD):
        pytest.fail("guard build missing: __graft_entry__.build() makes it")
    g = _run(GUARD)
    p = _run()
    guard = [ln for ln in g if ln.startswith("GUARD")]
    assert guard and guard[0].split()[1] == "0", guard
    assert [ln for ln in g if not ln.startswith("GUARD")] == p
