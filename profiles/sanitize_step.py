"""One small outer iteration per solver path, for compute-sanitizer (memcheck / racecheck /
synccheck): the 2-colour path with harmonic lanes (FD Jacobian, residual, linearized
residual, DF, the batched sweep with its last-CTA stopping rule), the level-scheduled
path (tets), and the explicit block-Jacobi arm.  usage: compute-sanitizer --tool memcheck
python profiles/sanitize_step.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402

for name, scale, workers, implicit in (("c2", 0.05, 3, True), ("c3", 0.04, 2, True), ("c1", 0.25, 1, False)):
    c = make_case(name, scale=scale, nh=2, workers=workers, implicit=implicit)
    s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
    e = s.outer_iteration()
    print(name, c.mesh.n, "nodes", "resid_mean", e["resid_mean"], flush=True)
