"""SPEC acceptance criterion 7 on the reference nozzle (tests/golden/nozzle_nx64_h2.npz):
FNLH (implicit, run to convergence) vs the time-accurate oracle (csrc/urans.cu) started from
the FNLH mean; per-harmonic relative L2 amplitude error over interior nodes, plus the
march's step count, dt, periods and the last period-to-period change.  Also runs the C1
configuration at reduced scale.  Usage: python profiles/urans_ac7.py"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import embed, forcing_triplets, line_mesh_from_ref, nozzle_from_golden, rel  # noqa: E402
from paper_2404_01407_b200 import urans  # noqa: E402
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402


def compare(name, g, m, max_iters):
    t0 = time.time()
    reason, hist = g.run_to_convergence()
    t_f = time.time() - t0
    mean_f, amps_f = g.state()
    t0 = time.time()
    ts = urans.unsteady_solve(g, mean_f, urans.OracleOptions(max_periods=4000))
    t_u = time.time() - t0
    mean_t, amps_t = urans.extract_harmonics(ts, g.omegas)
    errs = urans.compare_amplitudes(amps_f, amps_t, m)
    out = dict(case=name, nodes=m.n, fnlh=dict(reason=reason, iters=len(hist), wall_s=round(t_f, 2)),
               urans=dict(ts.info, wall_s=round(t_u, 2)), amp_rel_l2=[round(e[1], 5) for e in errs],
               mean_rel_l2=float(rel(mean_t, mean_f)))
    print(json.dumps(out), flush=True)


noz = nozzle_from_golden(os.path.join(ROOT, "tests", "golden", "nozzle_nx64_h2.npz"))
m = line_mesh_from_ref(noz)
m.ijk = np.stack([np.arange(noz.n), np.zeros(noz.n, np.int64), np.zeros(noz.n, np.int64)], axis=1)
forc = np.stack([forcing_triplets(f) for f in noz.forcing])
compare("nozzle nx64, 2 harmonics, amplitude 1e-3 (AC7)",
        FnlhSolver(m, dict(implicit=1, max_outer_iters=600, target_drop_orders=10.0), noz.omega, forc,
                   embed(noz.mean0, noz.n), pattern=noz.pattern(5)), m, 600)
c = make_case("c1", scale=0.5, nh=1)
c.scheme.update(max_outer_iters=400, target_drop_orders=8.0, linear_tol=1e-2, linear_max_iter=10)
compare("c1 at scale 0.5, 1 harmonic", FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0), c.mesh, 400)
