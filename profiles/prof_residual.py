"""Profiling driver: the C2 second-order residual (k_jst_prepass, k_face_flux,
k_node_gather) -- 5 warm-up evaluations then 10 profiled ones -- and the FD Jacobian."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import Discretization  # noqa: E402

c = make_case("c2", scale=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
d = Discretization(c.mesh)
for _ in range(15):
    d.residual(c.mean0, 2)
for _ in range(2):
    d.fd_jacobian(c.mean0, want_J=True)
