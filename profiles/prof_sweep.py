"""Profiling driver: C2 harmonic sweeps (the roofline kernel), optionally after one
pseudo-step (--step).  Default: the exact (bitwise) sweep; --onepass the one-pass
sweep; --all every variant.  Run under ncu with -k regex:k_rb to capture the sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200 import la  # noqa: E402
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1][0].isdigit() else 1.0
c = make_case("c2", scale=scale)
s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
if "--step" in sys.argv:
    s.outer_iteration()
names = {la.RB_EXACT: "exact", la.RB_EXACT_SPLIT: "exact-split", la.RB_ONEPASS: "one-pass"}
modes = list(names) if "--all" in sys.argv else [la.RB_ONEPASS if "--onepass" in sys.argv else la.RB_EXACT]
for mode in modes:
    la.set_rb_sweep(mode)
    s.time_sweeps(0, 3)
    print(names[mode], "sweep ms", s.time_sweeps(0, 20) / 20)
la.set_rb_sweep(la.RB_EXACT)
