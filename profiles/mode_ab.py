"""A/B of 2-colour sweep variants (fnlh_set_rb_sweep) on one solver, alternating within one
process: batched (all lanes) and single-lane sweep times.
usage: python profiles/mode_ab.py c4 8 0 3   (case, lanes, modes...)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200 import la  # noqa: E402
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402

name, P = sys.argv[1], int(sys.argv[2])
modes = [int(m) for m in sys.argv[3:]] or [0, 3]
c = make_case(name, workers=P)
s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
res = {m: ([], []) for m in modes}
for rnd in range(3):
    for m in modes:
        la.set_rb_sweep(m)
        if P > 1:
            s.time_sweeps_batch(P, 2)
            res[m][0].append(s.time_sweeps_batch(P, 10) / 10)
        s.time_sweeps(0, 2)
        res[m][1].append(s.time_sweeps(0, 10) / 10)
la.set_rb_sweep(0)
for m, (b, one) in res.items():
    print(f"{name} mode {m}: batched x{P} {min(b) if b else float('nan'):.4f} ms  single {min(one):.4f} ms", flush=True)
