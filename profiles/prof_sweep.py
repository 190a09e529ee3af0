"""Profiling driver: C2 (or --case cN) harmonic sweeps (the roofline kernel), optionally after one
pseudo-step (--step).  Default: the exact (bitwise) sweep; --onepass the one-pass
sweep; --all every variant; --batch P also times the batched sweep of P harmonic lanes
(workers = P).  Run under ncu with -k regex:k_rb to capture the sweep kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200 import la  # noqa: E402
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402

args = sys.argv[1:]
scale = float(args[0]) if args and args[0][0].isdigit() else 1.0
P = int(args[args.index("--batch") + 1]) if "--batch" in args else 1
case = args[args.index("--case") + 1] if "--case" in args else "c2"
kw = {"order": args[args.index("--order") + 1]} if "--order" in args else {}
c = make_case(case, scale=scale, workers=P, **kw)
s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
if "--step" in args:
    s.outer_iteration()
names = {la.RB_EXACT: "exact", la.RB_EXACT_SPLIT: "exact-split", la.RB_ONEPASS: "one-pass"}
names[la.RB_EDGE] = "edge-parallel"
names[la.RB_LANEWARP] = "lane-warp"
names[la.RB_STAGED] = "staged"
names[la.RB_ASTAGED] = "A-staged"
modes = list(names) if "--all" in args else [la.RB_ONEPASS if "--onepass" in args else la.RB_EXACT]
if "--mode" in args:
    modes = [int(args[args.index("--mode") + 1])]
for mode in modes:
    la.set_rb_sweep(mode)
    if "--only-batch" not in args:
        s.time_sweeps(0, 3)
        print(names[mode], "sweep ms", s.time_sweeps(0, 20) / 20)
    if P > 1:
        s.time_sweeps_batch(P, 3)
        t = s.time_sweeps_batch(P, 20) / 20
        print(f"  {names[mode]} batched x{P}: ms per batched sweep {t:.4f}, per harmonic sweep {t / P:.4f}")
la.set_rb_sweep(la.RB_EXACT)
