"""A/B timing of the harmonic sweep under runtime switches (environment variables read by
the library per solve), alternating the variants within one process so box-to-box and
drift effects cancel.  usage: python profiles/ab_sweep.py --case c4 --batch 8
    --var base: --var nopf:FNLH_RB_PF=0 ..."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="c4")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--sweeps", type=int, default=10)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--var", action="append", default=[])
a = ap.parse_args()
vars_ = []
for v in a.var or ["base:"]:
    name, _, env = v.partition(":")
    vars_.append((name, dict(kv.split("=") for kv in env.split(",") if kv)))
c = make_case(a.case, scale=a.scale, workers=a.batch)
s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
res = {n: [] for n, _ in vars_}
for r in range(a.rounds):
    for name, env in vars_:
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        if a.batch > 1:
            s.time_sweeps_batch(a.batch, 2)
            t = s.time_sweeps_batch(a.batch, a.sweeps) / a.sweeps
        else:
            s.time_sweeps(0, 2)
            t = s.time_sweeps(0, a.sweeps) / a.sweeps
        res[name].append(t)
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
for name, ts in res.items():
    print(f"{a.case} P={a.batch} {name:12s} ms/sweep min {min(ts):.4f}  all {' '.join(f'{t:.4f}' for t in ts)}")
