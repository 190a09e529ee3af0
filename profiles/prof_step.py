"""One outer iteration of a configuration as bench.py builds it (for ncu captures of the
non-sweep kernels).  usage: python profiles/prof_step.py [c4] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = make_case(name)
c = make_case(name, workers=min(len(c.omegas), 8))
s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
for _ in range(steps):
    print(s.outer_iteration()["resid_mean"], flush=True)
