"""The explicit arm continued from a saved (mean, amps) state equals the uninterrupted run bit for
bit (profiles/mg_compare.py --checkpoint relies on it).  Exit code 0 when equal."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402


def mk():
    c = make_case("c5", scale=0.12, nh=5, implicit=False)
    c.scheme.update(dict(implicit=0, sigma_cfl=1.0))
    return FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)


a = mk()
ra = [(e["resid_mean"], e["rz"]) for e in (a.outer_iteration() for _ in range(8))]
b = mk()
rb = [(e["resid_mean"], e["rz"]) for e in (b.outer_iteration() for _ in range(4))]
mean, amps = b.state()
c = mk()
c.set_state(mean, amps)
rb += [(e["resid_mean"], e["rz"]) for e in (c.outer_iteration() for _ in range(4))]
print("equal" if ra == rb else f"DIFFERENT\n{ra}\n{rb}")
sys.exit(0 if ra == rb else 1)
