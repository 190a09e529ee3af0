"""Profiling driver: one C2 pseudo-step then 10 harmonic sweeps (the roofline kernel).
Run under ncu with -k regex:k_rb_colour to capture the fused sweep kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1][0].isdigit() else 1.0
c = make_case("c2", scale=scale)
s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
if "--step" in sys.argv:
    s.outer_iteration()
print("sweep ms", s.time_sweeps(0, 10) / 10)
