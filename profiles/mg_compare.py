"""Implicit FNLH vs explicit RK(5,3) single grid vs explicit + FAS V-cycle (2, 3 levels):
outer iterations and device seconds to drop the mean and harmonic residuals by `drop`
orders (run_to_convergence semantics, driver.cpp:335-379) on one seeded configuration.
The paper's comparison (PAPER.md: implicit 7-10x faster than explicit multigrid) restated
on the synthetic C2 geometry at reduced size.  Usage: python profiles/mg_compare.py
[--scale 0.25] [--drop 3] [--max 4000] [--cfl-explicit 1.0]"""
import argparse
import json
import sys
import time
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.solver import FnlhSolver  # noqa: E402


STOP_MEAN = False
CKPT, CKPT_AFTER = "", 3300.0


def run(name, scale, nh, scheme_over, drop, cap):
    c = make_case(name, scale=scale, nh=nh, implicit=scheme_over.get("implicit", 1) == 1)
    c.scheme.update(scheme_over)
    c.scheme["target_drop_orders"] = drop
    c.scheme["max_outer_iters"] = cap
    t0 = time.time()
    g = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
    setup = time.time() - t0
    t0 = time.time()
    try:
        if STOP_MEAN:
            # the same loop entry by entry (as cli.py drives it), left as soon as the MEAN residual
            # has dropped by `drop` orders -- for arms whose harmonic residual never gets there
            hist, reason = [], "iteration-cap"
            it0, s0, t_call = 0, 0.0, time.time()
            if CKPT and os.path.exists(CKPT + ".npz"):
                # continue a run a previous call had to leave (one gpurun call is at most 3,600 s):
                # the explicit scheme's whole state is (mean, amps); device seconds add up
                import numpy as np
                z = np.load(CKPT + ".npz")
                g.set_state(z["mean"], z["amps"])
                hist = [dict(iter=int(a), resid_mean=float(b), rz=float(c_), seconds=float(d)) for a, b, c_, d in z["hist"]]
                it0, s0 = len(hist), hist[-1]["seconds"]
                print(f"# resumed from {CKPT}.npz at iteration {it0}, {s0:.1f} device s", flush=True)
            for _ in range(it0, cap):
                e = g.outer_iteration()
                hist.append(dict(iter=len(hist), resid_mean=e["resid_mean"], rz=e["rz"], seconds=s0 + e["seconds"]))
                e = hist[-1]
                if CKPT and (time.time() - t_call > CKPT_AFTER):
                    import numpy as np
                    mean, amps = g.state()
                    np.savez(CKPT, mean=mean, amps=amps,
                             hist=np.array([[h["iter"], h["resid_mean"], h["rz"], h["seconds"]] for h in hist]))
                    print(f"# checkpoint at iteration {len(hist)}, {e['seconds']:.1f} device s -> {CKPT}.npz", flush=True)
                    reason = "checkpointed"
                    break
                if len(hist) % 2000 == 0:
                    print(f"# {len(hist)} iterations, {e['seconds']:.1f} s, mean residual {e['resid_mean']:.4e} "
                          f"({hist[0]['resid_mean'] / e['resid_mean']:.3e}x down), rz {e['rz']:.4e}", flush=True)
                if e["resid_mean"] <= hist[0]["resid_mean"] * 10.0 ** (-drop):
                    reason = "mean-target-drop"
                    break
        else:
            reason, hist = g.run_to_convergence()
    except Exception as ex:  # a non-divergence error ends the run (propagates in the reference)
        return dict(n=c.mesh.n, levels=g.levels(), reason=f"error: {ex}", iters=None, device_s=None)
    wall = time.time() - t0
    last = hist[-1] if hist else {}
    out = dict(n=c.mesh.n, levels=g.levels(), reason=reason, iters=len(hist), device_s=last.get("seconds", 0.0),
               wall_s=wall, setup_s=setup, r0=hist[0]["resid_mean"] if hist else None,
               r_end=last.get("resid_mean"), rz0=hist[0]["rz"] if hist else None, rz_end=last.get("rz"))
    # first outer iteration (1-based) and device seconds at which each residual had dropped
    # by `drop` orders from its first-iteration value (run_to_convergence's test, per field)
    for key, name in (("resid_mean", "mean"), ("rz", "rz")):
        if not hist:
            break
        tgt = hist[0][key] * 10.0 ** (-drop)
        hit = next((e for e in hist if e[key] <= tgt), None)
        out[f"{name}_drop_iter"] = hit["iter"] + 1 if hit else None
        out[f"{name}_drop_s"] = hit["seconds"] if hit else None
        # every whole order on the way: [orders, iteration, device seconds]
        orders = []
        for o in range(1, int(drop) + 1):
            h = next((e for e in hist if e[key] <= hist[0][key] * 10.0 ** (-o)), None)
            if h is None:
                break
            orders.append([o, h["iter"] + 1, round(h["seconds"], 3)])
        out[f"{name}_orders"] = orders
        # the lowest value reached and where, and how far the run climbed back from it
        # (a residual that rises again after its minimum: the run is diverging slowly)
        k_min = min(range(len(hist)), key=lambda q: hist[q][key])
        out[f"{name}_min"] = [hist[k_min][key], k_min + 1, round(hist[k_min]["seconds"], 3)]
        out[f"{name}_end_over_min"] = hist[-1][key] / max(hist[k_min][key], 1e-300)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="c2")
    ap.add_argument("--scale", type=float, default=0.25)
    ap.add_argument("--nh", type=int, default=2)
    ap.add_argument("--drop", type=float, default=3.0)
    ap.add_argument("--max", type=int, default=4000)
    ap.add_argument("--cfl-explicit", type=float, default=1.0)
    ap.add_argument("--max-implicit", type=int, default=0, help="iteration cap of the implicit arm (0: --max)")
    ap.add_argument("--arms", default="implicit,explicit_1grid,explicit_mg2,explicit_mg3")
    ap.add_argument("--stop-mean", action="store_true", help="leave an arm once its mean residual reached the drop")
    ap.add_argument("--checkpoint", default="", help="with --stop-mean: resume from / save to this path (.npz)")
    ap.add_argument("--checkpoint-after", type=float, default=3300.0, help="wall seconds after which to save and leave")
    a = ap.parse_args()
    global STOP_MEAN, CKPT, CKPT_AFTER
    STOP_MEAN, CKPT, CKPT_AFTER = a.stop_mean, a.checkpoint, a.checkpoint_after
    arms = {
        "implicit": dict(implicit=1, workers=a.nh),
        "explicit_1grid": dict(implicit=0, sigma_cfl=a.cfl_explicit),
        "explicit_mg2": dict(implicit=0, sigma_cfl=a.cfl_explicit, mg_levels=2),
        "explicit_mg3": dict(implicit=0, sigma_cfl=a.cfl_explicit, mg_levels=3),
    }
    out = {}
    for k, v in arms.items():
        if k not in a.arms.split(","):
            continue
        cap = a.max_implicit if (k == "implicit" and a.max_implicit) else a.max
        out[k] = run(a.case, a.scale, a.nh, v, a.drop, cap)
        print(k, json.dumps(out[k]), flush=True)
    print(json.dumps(dict(case=a.case, scale=a.scale, nh=a.nh, drop=a.drop, arms=out)))


if __name__ == "__main__":
    main()
