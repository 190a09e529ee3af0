"""Two small outer iterations per solver path, run against the guard build of the library
(FNLH_B200_LIB=.../libfnlh_b200_guard.so, tests/test_gpu_guard.py): the 2-colour path with
harmonic lanes (FD Jacobian, residual, linearized residual, DF, the batched sweep with its
last-CTA stopping rule), the level-scheduled path (tets), the explicit block-Jacobi arm, and
the persistent operator handles.  Prints every residual (repr) and, in a guard build, the
overwritten guard bytes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402

import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402

from paper_2404_01407_b200 import la  # noqa: E402
from paper_2404_01407_b200._lib import lib  # noqa: E402

for name, scale, workers, implicit in (("c2", 0.05, 3, True), ("c3", 0.04, 2, True), ("c1", 0.25, 1, False),
                                       ("c2", 0.05, 1, True)):
    c = make_case(name, scale=scale, nh=2, workers=workers, implicit=implicit)
    s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
    for _ in range(2):
        e = s.outer_iteration()
        print("STEP", name, workers, repr(e["resid_mean"]), repr(e["rz"]), flush=True)
    del s
c = make_case("c2", scale=0.05)
pat = c.mesh.pattern()
rng = np.random.default_rng(3)
A = rng.standard_normal((len(pat["col_idx"]), 5, 5)) * 0.1
A[pat["diag_idx"]] += 4 * np.eye(5)
for rb in (True, False):
    la.set_red_black(rb)
    L = la.Lhs(la.Pattern.from_dict(pat), A.reshape(-1))
    w = la.Ilu(L, True)
    w.factorize(rng.uniform(0.5, 2.0, c.mesh.n))
    x, rep = w.solve(rng.standard_normal(c.mesh.n * 5) + 0j, 1e-3, 4)
    print("HANDLES", rb, repr(float(np.abs(x).sum())), rep[0], flush=True)
    del w, L
la.set_red_black(True)
bad, blocks = C.c_longlong(), C.c_longlong()
if lib().fnlh_guard_check(C.byref(bad), C.byref(blocks)) == 0:
    print("GUARD", bad.value, blocks.value, flush=True)
