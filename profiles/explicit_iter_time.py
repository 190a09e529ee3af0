"""Device seconds per explicit RK(5,3) outer iteration at full C5 size with workers = 1 and 5 (the
tet path runs its harmonics one after the other: 0.141 s either way).  usage: python profiles/explicit_iter_time.py"""
import sys, os, time
sys.path.insert(0, os.getcwd())
from paper_2404_01407_b200.cases import make_case
from paper_2404_01407_b200.solver import FnlhSolver
for w in (1, 5):
    c = make_case("c5", scale=1.0, nh=5, implicit=False, workers=w)
    c.scheme.update(dict(implicit=0, sigma_cfl=1.0, workers=w))
    g = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
    for _ in range(5): g.outer_iteration()
    e0 = g.outer_iteration()
    for _ in range(40): e = g.outer_iteration()
    print("workers", w, "lanes", g.lanes(), "s/iter", (e["seconds"] - e0["seconds"]) / 40, "resid", e["resid_mean"], flush=True)
    del g
