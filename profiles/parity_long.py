"""Full-size, full-length parity of the outer iteration against the CPU restatement (whose
linear algebra is bitwise the reference's): BASELINE C1 (20 pseudo-steps) and C2 (50), the
device path as bench.py runs it (C2: 3 harmonic lanes), the restatement with the
reference's harmonic worker threads.  The device solver runs as bench.py builds it:
workers = min(N_h, 8) harmonic lanes.  Prints per-step relative differences of the mean and
harmonic residual norms, the linear-iteration counts, and the final state difference.
Usage: python profiles/parity_long.py [c1 c2 c3:2 c4:1:3 ...]   (name[:steps[:oracle
workers]], default the BASELINE step count and one worker per harmonic)"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle  # noqa: E402
from paper_2404_01407_b200._lib import pow_mode  # noqa: E402
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


for arg in (sys.argv[1:] or ["c1", "c2"]):
    name, _, rest = arg.partition(":")
    k, _, w = rest.partition(":")  # name[:steps[:oracle workers]] (C4: each worker holds 24 GB)
    c = make_case(name)
    c = make_case(name, workers=min(len(c.omegas), 8))  # the bench's harmonic lanes
    c.pseudo_steps = int(k) if k else c.pseudo_steps
    nw = int(w) if w else min(len(c.omegas), os.cpu_count() or 1)
    g = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
    o = Oracle(pow_mode=pow_mode(), workers=nw).solver(c.mesh, c.mesh.pattern(), c.scheme,
                                                                         c.omegas, c.forcing, c.mean0)
    worst_m = worst_z = 0.0
    t0 = time.time()
    for it in range(c.pseudo_steps):
        eg, eo = g.outer_iteration(), o.outer_iteration()
        dm = abs(eg["resid_mean"] / eo["resid_mean"] - 1)
        dz = abs(eg["rz"] / eo["rz"] - 1) if eo["rz"] else 0.0
        worst_m, worst_z = max(worst_m, dm), max(worst_z, dz)
        print(f"{name} step {it + 1:3d} resid_mean {eg['resid_mean']:.6e} rel {dm:.2e}  R_z {eg['rz']:.6e} rel {dz:.2e}",
              flush=True)
    mg, ag = g.state()
    mo, ao = o.state()
    same_iters = [r[0] for r in g.reports()] == [r[0] for r in o.reports()]
    print(json.dumps(dict(case=name, nodes=c.mesh.n, steps=c.pseudo_steps, device_lanes=g.lanes(), oracle_workers=nw, max_rel_resid_mean=worst_m,
                          max_rel_rz=worst_z, final_mean_rel=rel(mg, mo), final_amps_rel=rel(ag, ao),
                          identical_linear_iteration_counts=same_iters, wall_s=round(time.time() - t0, 1))),
          flush=True)
