"""Batched harmonic sweep time vs lane count P at one configuration (per batched sweep and
per harmonic), the algorithmic bytes of each (bench.rb_sweep_bytes) and the HBM fraction:
which P the product should default to.  usage: python profiles/lanes_sweep.py c4"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import peaks, rb_sweep_bytes  # noqa: E402
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
c = make_case(name, workers=8)
s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
info = s.info()
n, b = c.mesh.n, c.mesh.b
E = (len(c.mesh.pattern()["col_idx"]) - n) // 2
peak, _ = peaks()
rows = []
for P in [1, 2, 3, 4, 5, 6, 7, 8]:
    if P == 1:
        s.time_sweeps(0, 2)
        ms = s.time_sweeps(0, 10) / 10
    else:
        s.time_sweeps_batch(P, 2)
        ms = s.time_sweeps_batch(P, 10) / 10
    by = rb_sweep_bytes(n, info["n0"], E, b, P)
    rows.append(dict(P=P, ms=ms, ms_per_harmonic=ms / P, GBps=by / ms / 1e6, frac=by / ms / 1e6 / peak))
    print(json.dumps(rows[-1]), flush=True)
