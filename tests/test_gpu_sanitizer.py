"""compute-sanitizer over one small outer iteration of every solver path
(profiles/sanitize_step.py): memcheck (out-of-bounds / misaligned accesses, including the
guard-free packed layouts), racecheck (shared-memory hazards, e.g. the colour-0 park and the
CTA reductions) and synccheck (barrier use of the last-CTA stopping rule) must report no
errors."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.fail("compute-sanitizer not found")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20", "python",
                        os.path.join(ROOT, "profiles", "sanitize_step.py")], capture_output=True, text=True,
                       timeout=1800, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
