"""Command-line entry point (SPEC.md cli module): run / oracle / compare / bench with the
machine-readable outputs the specification lists -- a fully materialized manifest, the
convergence CSV (iter, resid_mean, resid_h0..h{N_h-1}, R_z, seconds, WU), optional
final-field CSVs and a key-value summary.  The reference specifies these but ships no
CLI; the solver underneath is the device FnlhSolver.

    python -m paper_2404_01407_b200 run c2 --max-iters 50 --out runs/c2
    python -m paper_2404_01407_b200 run case.cfg --mode explicit --mg-levels 3
    python -m paper_2404_01407_b200 compare runs/a runs/b --bound 1e-8
    python -m paper_2404_01407_b200 oracle c1 --scale 0.5 --harmonics 1 --out runs/c1_oracle
    python -m paper_2404_01407_b200 bench memory-audit

Config files are plain-text `key = value` lines (# comments); keys: case (c1..c5),
scale, harmonics, mode (implicit|explicit), cfl, eps, tol, sweeps, mg_levels,
partitions, workers, target_drop, max_iters.  Exit codes of `run`: 0 target-drop,
3 iteration-cap, 4 divergence, 2 usage / configuration errors.
"""
from __future__ import annotations

import argparse
import csv
import os
import sys
import time

import numpy as np

EXIT = {"target-drop": 0, "iteration-cap": 3, "divergence": 4}
KEYS = {"case": str, "scale": float, "harmonics": int, "mode": str, "cfl": float, "eps": float, "tol": float,
        "sweeps": int, "mg_levels": int, "partitions": int, "workers": int, "target_drop": float, "max_iters": int}
REQUIRED = ("case",)


class ConfigParseError(ValueError):
    pass


def parse_config(text: str, source: str = "<config>") -> dict:
    """`key = value` lines; diagnostics name the line and the key."""
    out = {}
    for ln, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigParseError(f"{source}:{ln}: expected 'key = value', got {raw.strip()!r}")
        k, v = (t.strip() for t in line.split("=", 1))
        if k not in KEYS:
            raise ConfigParseError(f"{source}:{ln}: unknown key {k!r}")
        try:
            out[k] = KEYS[k](v)
        except ValueError:
            raise ConfigParseError(f"{source}:{ln}: key {k!r}: cannot parse {v!r} as {KEYS[k].__name__}") from None
    for k in REQUIRED:
        if k not in out:
            raise ConfigParseError(f"{source}: missing required key {k!r}")
    return out


def resolve(args) -> dict:
    """Materialize every setting: config file (or case name), then command-line overrides."""
    from .cases import SPECS
    if os.path.exists(args.config):
        with open(args.config) as f:
            cfg = parse_config(f.read(), args.config)
    else:
        cfg = {"case": args.config}
    for k in KEYS:
        v = getattr(args, k, None)
        if v is not None:
            cfg[k] = v
    if cfg["case"] not in SPECS:
        raise ConfigParseError(f"case: unknown case id {cfg['case']!r} (expected one of {sorted(SPECS)})")
    spec = SPECS[cfg["case"]]
    mode = cfg.get("mode", "implicit")
    if mode not in ("implicit", "explicit"):
        raise ConfigParseError(f"mode: expected implicit or explicit, got {mode!r}")
    nh = cfg.get("harmonics", spec["nh"])
    r = dict(case=cfg["case"], scale=cfg.get("scale", 1.0), harmonics=nh, mode=mode,
             cfl=cfg.get("cfl", spec["sigma"] if mode == "implicit" else -1.0), eps=cfg.get("eps", 0.6),
             tol=cfg.get("tol", spec["tol"]), sweeps=cfg.get("sweeps", spec["max_iter"]),
             mg_levels=cfg.get("mg_levels", 1), partitions=cfg.get("partitions", 1),
             workers=cfg.get("workers", max(1, min(nh, 8))), target_drop=cfg.get("target_drop", 8.0),
             max_iters=cfg.get("max_iters", spec["steps"]))
    if r["mg_levels"] > 1 and mode == "implicit":
        raise ConfigParseError("mg_levels: multigrid is available for the explicit scheme only")
    if r["cfl"] <= 0:  # per-mode default (driver.hpp:33-41)
        r["cfl"] = 50.0 if mode == "implicit" else 2.0
    return r


def build_solver(r: dict):
    from .cases import make_case
    from .solver import FnlhSolver
    c = make_case(r["case"], scale=r["scale"], nh=r["harmonics"], implicit=r["mode"] == "implicit",
                  workers=r["workers"])
    if r["partitions"] > 1:
        # the reference's contiguous_partitions (mesh.cpp:62-67) split its 1D node order into
        # spatial ranges; the 3D analogue on the colour-major order is axial slabs
        # (index ranges would put whole colours in different partitions)
        i = c.mesh.ijk[:, 0]
        c.mesh.partition = ((i * r["partitions"]) // (int(i.max()) + 1)).astype(np.int32)
    c.scheme.update(sigma_cfl=r["cfl"], eps_relax=r["eps"], linear_tol=r["tol"], linear_max_iter=r["sweeps"],
                    target_drop_orders=r["target_drop"], max_outer_iters=r["max_iters"], mg_levels=r["mg_levels"],
                    workers=r["workers"])
    return c, FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)


def t_ref() -> float:
    from ._lib import lib
    import ctypes as C
    lib().fnlh_normalization_kernel_seconds.restype = C.c_double
    return float(lib().fnlh_normalization_kernel_seconds())


def run_loop(g, r, on_entry=None):
    """run_to_convergence (driver.cpp:335-379) driven entry by entry (the CSV needs every
    harmonic's residual per iteration)."""
    from ._lib import FnlhError
    drop = 10.0 ** (-r["target_drop"])
    hist, reason, msg = [], "iteration-cap", ""
    r1_mean = r1_rz = floor = 0.0
    for it in range(r["max_iters"]):
        try:
            e = g.outer_iteration()
        except FnlhError as ex:
            if ex.kind != "DivergenceError":
                raise
            reason, msg = "divergence", str(ex)
            break
        hist.append(e)
        if on_entry:
            on_entry(e)
        if it == 0:
            r1_mean, r1_rz = e["resid_mean"], (e["rz"] if e["has_rz"] else 0.0)
            floor = 1e-16 * max(r1_mean, r1_rz)
        mean_ok = e["resid_mean"] <= max(r1_mean * drop, floor)
        rz_ok = not e["has_rz"] or e["rz"] <= max(r1_rz * drop, floor)
        if mean_ok and rz_ok:
            reason = "target-drop"
            break
    return hist, reason, msg


def write_kv(path, items):
    with open(path, "w") as f:
        for k, v in items:
            f.write(f"{k} = {v}\n")


def read_kv(path):
    out = {}
    with open(path) as f:
        for line in f:
            if "=" in line:
                k, v = line.split("=", 1)
                out[k.strip()] = v.strip()
    return out


def write_manifest(out, r, c, tr, extra=()):
    write_kv(os.path.join(out, "manifest.txt"),
             [("case", r["case"]), ("description", c.description), ("nodes", c.mesh.n), ("block_size", c.mesh.b)] +
             [(k, r[k]) for k in ("scale", "harmonics", "mode", "cfl", "eps", "tol", "sweeps", "mg_levels",
                                  "partitions", "workers", "target_drop", "max_iters")] +
             [("omegas", " ".join(repr(float(w)) for w in c.omegas)), ("output_dir", os.path.abspath(out)),
              ("t_ref_seconds", repr(tr)), ("data", "synthetic (seeded, cases.py)")] + list(extra))


def write_fields(out, mean, amps, b):
    np.savetxt(os.path.join(out, "field_mean.csv"), np.asarray(mean).reshape(-1, b), delimiter=",",
               header=",".join(f"w{k}" for k in range(b)), comments="", fmt="%.17g")
    for h in range(len(amps)):
        a = np.asarray(amps[h]).reshape(-1, b)
        np.savetxt(os.path.join(out, f"field_h{h}.csv"), np.concatenate([a.real, a.imag], axis=1), delimiter=",",
                   header=",".join([f"re{k}" for k in range(b)] + [f"im{k}" for k in range(b)]), comments="",
                   fmt="%.17g")


def cmd_oracle(args) -> int:
    """SPEC oracle_urans through the CLI: run_to_convergence, then the time-accurate march
    (urans.unsteady_solve) from the converged mean.  Writes the oracle's fields (time mean,
    DFT amplitudes) in the run layout, so `compare <run dir> <oracle dir>` applies, plus
    amplitude_errors.csv (compare_amplitudes: interior nodes) against the FNLH fields of
    the same run.  Exit 0, or 3 when either the FNLH run or the march hits its cap, 4 on
    divergence."""
    from . import urans
    from ._lib import FnlhError
    r = resolve(args)
    out = args.out or os.path.join("runs", f"{r['case']}_oracle")
    os.makedirs(out, exist_ok=True)
    tr = t_ref()
    c, g = build_solver(r)
    hist, reason, msg = run_loop(g, r)
    if reason == "divergence":
        print(f"oracle: the FNLH run diverged ({msg})", file=sys.stderr)
        return EXIT[reason]
    mean_f, amps_f = g.state()
    opt = urans.OracleOptions(samples_per_period=args.samples, cfl=args.oracle_cfl, max_periods=args.max_periods)
    t0 = time.time()
    code = 0
    try:
        ts = urans.unsteady_solve(g, mean_f, opt)
    except FnlhError as ex:
        if ex.kind != "NonConvergenceError":
            raise
        ts, code = ex.timeseries, 3
        print(f"oracle: {ex}", file=sys.stderr)
    wall = time.time() - t0
    mean_t, amps_t = urans.extract_harmonics(ts, g.omegas)
    write_manifest(out, r, c, tr, [("kind", "oracle_urans")])
    write_fields(out, mean_t, amps_t, c.mesh.b)
    errs = urans.compare_amplitudes(amps_f, amps_t, c.mesh)
    with open(os.path.join(out, "amplitude_errors.csv"), "w") as f:
        f.write("harmonic,omega,rel_l2_interior\n")
        for (l, e), om in zip(errs, g.omegas):
            f.write(f"{l},{float(om)!r},{e!r}\n")
    write_kv(os.path.join(out, "summary.txt"),
             [("case", r["case"]), ("fnlh_reason", reason), ("fnlh_iterations", len(hist)),
              ("samples", ts.info["samples"]), ("steps_per_period", ts.info["steps_per_period"]),
              ("dt", repr(ts.info["dt"])), ("periods", ts.info["periods"]),
              ("last_change", repr(ts.info["last_change"])), ("march_wall_seconds", f"{wall:.3f}"),
              ("periodic", int(code == 0))] + [(f"amp_error_h{l}", repr(e)) for l, e in errs])
    for l, e in errs:
        print(f"harmonic {l}: FNLH vs time-accurate relative L2 (interior) {e:.3e}")
    print(f"-> {out}")
    if code == 0 and reason != "target-drop":
        code = EXIT[reason]
    return code


def cmd_run(args) -> int:
    r = resolve(args)
    out = args.out or os.path.join("runs", f"{r['case']}_{r['mode']}")
    os.makedirs(out, exist_ok=True)
    tr = t_ref()
    t0 = time.time()
    c, g = build_solver(r)
    setup = time.time() - t0
    write_manifest(out, r, c, tr)
    nh = r["harmonics"]
    fcsv = open(os.path.join(out, "convergence.csv"), "w", newline="")
    w = csv.writer(fcsv)
    w.writerow(["iter", "resid_mean"] + [f"resid_h{h}" for h in range(nh)] + ["R_z", "seconds", "WU"])

    def row(e):
        wu = r["workers"] * e["seconds"] / tr
        w.writerow([e["iter"], repr(e["resid_mean"])] + [repr(float(x)) for x in e["resid_h"]] +
                   [repr(e["rz"]), repr(e["seconds"]), repr(wu)])
        fcsv.flush()

    hist, reason, msg = run_loop(g, r, row)
    fcsv.close()
    if args.fields:
        write_fields(out, *g.state(), c.mesh.b)
    last = hist[-1] if hist else dict(resid_mean=float("nan"), rz=float("nan"), seconds=0.0)
    write_kv(os.path.join(out, "summary.txt"),
             [("case", r["case"]), ("mode", r["mode"]), ("sigma_cfl", r["cfl"]), ("mg_levels", r["mg_levels"]),
              ("reason", reason), ("divergence_message", msg), ("iterations", len(hist)),
              ("resid_mean", repr(last["resid_mean"])), ("R_z", repr(last["rz"])),
              ("seconds", repr(last["seconds"])), ("WU", repr(r["workers"] * last["seconds"] / tr)),
              ("t_ref_seconds", repr(tr)), ("peak_lhs_bytes", g.lhs_bytes()), ("setup_seconds", f"{setup:.3f}"),
              ("exit_code", EXIT[reason])])
    print(f"{r['case']} {r['mode']}: {reason} after {len(hist)} outer iterations, "
          f"resid_mean {last['resid_mean']:.3e}, R_z {last['rz']:.3e}, {last['seconds']:.3f} s -> {out}")
    return EXIT[reason]


def cmd_compare(args) -> int:
    """Per-field relative L2 error between two runs' final fields (same case id)."""
    ma, mb = read_kv(os.path.join(args.a, "manifest.txt")), read_kv(os.path.join(args.b, "manifest.txt"))
    if (ma.get("case"), ma.get("scale"), ma.get("harmonics")) != (mb.get("case"), mb.get("scale"), mb.get("harmonics")):
        print(f"compare: case mismatch ({ma.get('case')} scale {ma.get('scale')} vs {mb.get('case')} "
              f"scale {mb.get('scale')})", file=sys.stderr)
        return 2
    rows, ok = [], True
    names = ["field_mean.csv"] + [f"field_h{h}.csv" for h in range(int(ma.get("harmonics", 0)))]
    for nm in names:
        pa, pb = os.path.join(args.a, nm), os.path.join(args.b, nm)
        if not (os.path.exists(pa) and os.path.exists(pb)):
            print(f"compare: {nm} missing (run with --fields)", file=sys.stderr)
            return 2
        xa, xb = np.loadtxt(pa, delimiter=",", skiprows=1), np.loadtxt(pb, delimiter=",", skiprows=1)
        err = float(np.linalg.norm(xa - xb) / max(np.linalg.norm(xb), 1e-300))
        passed = err <= args.bound
        ok &= passed
        rows.append((nm, err, passed))
    out = args.out or os.path.join(args.a, "compare.txt")
    with open(out, "w") as f:
        f.write(f"# {args.a} vs {args.b}, bound {args.bound:g}\nfield,rel_l2_error,pass\n")
        for nm, err, p in rows:
            f.write(f"{nm},{err!r},{int(p)}\n")
    for nm, err, p in rows:
        print(f"{nm:16s} {err:.3e} {'pass' if p else 'FAIL'}")
    return 0 if ok else 1


def cmd_bench(args) -> int:
    suite = args.suite
    out = args.out or f"bench_{suite}.csv"
    tr = t_ref()
    ns = argparse.Namespace(**{k: None for k in KEYS})
    ns.config = args.case
    rows = []
    if suite == "memory-audit":  # SPEC AC3: LHS bytes identical for N_h = 1, 2, 4, 8
        for nh in (1, 2, 4, 8):
            ns.harmonics, ns.scale, ns.workers = nh, args.scale, 1
            _, g = build_solver(resolve(ns))
            rows.append(dict(harmonics=nh, peak_lhs_bytes=g.lhs_bytes()))
        same = len({r_["peak_lhs_bytes"] for r_ in rows}) == 1
        print("memory-audit:", "LHS bytes independent of N_h" if same else "LHS bytes DEPEND on N_h")
    elif suite in ("convergence-ordering", "partition-sweep", "wu-report"):
        if suite == "convergence-ordering":
            arms = [("implicit", dict(mode="implicit")), ("explicit-4MG", dict(mode="explicit", mg_levels=4)),
                    ("explicit-1MG", dict(mode="explicit", mg_levels=1))]
        elif suite == "partition-sweep":
            arms = [(f"implicit-P{p}", dict(mode="implicit", partitions=p)) for p in (1, 2, 4, 8)]
        else:
            arms = [("implicit", dict(mode="implicit"))]
        for name, over in arms:
            nsx = argparse.Namespace(**vars(ns))
            nsx.scale, nsx.max_iters, nsx.target_drop = args.scale, args.max_iters, args.target_drop
            nsx.cfl = args.cfl_explicit if over["mode"] == "explicit" else None
            for k, v in over.items():
                setattr(nsx, k, v)
            r = resolve(nsx)
            _, g = build_solver(r)
            try:
                hist, reason, _ = run_loop(g, r)
            except Exception as ex:  # a non-divergence error ends the arm (it propagates in the reference)
                hist, reason = [], f"error: {str(ex).split(':')[0]}"
            hist = hist or []
            sec = hist[-1]["seconds"] if hist else 0.0
            rows.append(dict(scheme=name, reason=reason, outer_iterations=len(hist), seconds=sec,
                             WU=r["workers"] * sec / tr, peak_lhs_bytes=g.lhs_bytes()))
            print(f"{name:14s} {reason:14s} {len(hist):6d} iterations {sec:9.3f} s")
    else:
        print(f"bench: unknown suite {suite!r}", file=sys.stderr)
        return 2
    with open(out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
    print(f"-> {out} (t_ref {tr:.4f} s)")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2404_01407_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    pr = sub.add_parser("run", help="run_to_convergence with manifest / convergence CSV / summary")
    pr.add_argument("config", help="case id (c1..c5) or a key = value config file")
    pr.add_argument("--mode", choices=["implicit", "explicit"])
    pr.add_argument("--cfl", type=float)
    pr.add_argument("--eps", type=float)
    pr.add_argument("--tol", type=float)
    pr.add_argument("--sweeps", type=int)
    pr.add_argument("--mg-levels", dest="mg_levels", type=int)
    pr.add_argument("--harmonics", type=int)
    pr.add_argument("--partitions", type=int)
    pr.add_argument("--workers", type=int)
    pr.add_argument("--target-drop", dest="target_drop", type=float)
    pr.add_argument("--max-iters", dest="max_iters", type=int)
    pr.add_argument("--scale", type=float)
    pr.add_argument("--out")
    pr.add_argument("--fields", action="store_true", help="write the final fields as CSV")
    po = sub.add_parser("oracle", help="FNLH run, then the time-accurate reference march (SPEC oracle_urans)")
    po.add_argument("config")
    for k in ("--cfl", "--eps", "--tol", "--scale"):
        po.add_argument(k, type=float)
    for k, d in (("--sweeps", "sweeps"), ("--harmonics", "harmonics"), ("--workers", "workers"),
                 ("--max-iters", "max_iters"), ("--mg-levels", "mg_levels"), ("--partitions", "partitions")):
        po.add_argument(k, dest=d, type=int)
    po.add_argument("--mode", choices=["implicit", "explicit"])
    po.add_argument("--target-drop", dest="target_drop", type=float)
    po.add_argument("--samples", type=int, default=32, help="samples per period (raised to 4 l_max + 2)")
    po.add_argument("--oracle-cfl", dest="oracle_cfl", type=float, default=0.7)
    po.add_argument("--max-periods", dest="max_periods", type=int, default=200)
    po.add_argument("--out")
    pc = sub.add_parser("compare", help="per-field error report between two runs")
    pc.add_argument("a")
    pc.add_argument("b")
    pc.add_argument("--bound", type=float, default=1e-8)
    pc.add_argument("--out")
    pb = sub.add_parser("bench", help="benchmark suites")
    pb.add_argument("suite", help="memory-audit | convergence-ordering | partition-sweep | wu-report")
    pb.add_argument("--case", default="c1")
    pb.add_argument("--scale", type=float, default=0.5)
    pb.add_argument("--max-iters", dest="max_iters", type=int, default=200)
    pb.add_argument("--target-drop", dest="target_drop", type=float, default=3.0)
    pb.add_argument("--cfl-explicit", dest="cfl_explicit", type=float, default=0.5)
    pb.add_argument("--out")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "run":
            return cmd_run(a)
        if a.cmd == "compare":
            return cmd_compare(a)
        if a.cmd == "oracle":
            return cmd_oracle(a)
        return cmd_bench(a)
    except ConfigParseError as ex:
        print(f"error: {ex}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
