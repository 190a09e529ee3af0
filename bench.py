#!/usr/bin/env python
"""Benchmark of the FNLH implicit pseudo-time hot path on B200.

Workload: BASELINE.json configs[1] (C2): annular hex sector 128x64x48, 410,865 nodes,
5 conservative variables, 3 harmonics, implicit scheme (tol 1e-2, <= 10 sweeps).
A step is one pseudo-step (FnlhSolver::outer_iteration, driver.cpp:157-333): FD
Jacobian, A5 + real ILU(0), per harmonic complex ILU(0) + RK(5,3) with the
linearized residual and ILU-Richardson sweeps, DF, mean RK(5,3).

  value = block-row updates performed in the timed steps (sum over every stage solve
          of iterations x N) / device time of the timed steps, all ranks
  e2e   = same through the C ABI with host buffers (state uploaded and downloaded
          every step)
  roofline = the harmonic relaxation sweep (smoothed_solve iteration), algorithmic
          bytes of the stored-factor ILU formula / measured sweep time

Multi-GPU (--gpus N under torchrun): independent replicas (one C2 instance per
rank, no collective), "scaling": "weak".  --impl reference: the CPU path (oracle
restatement whose generic layers are bitwise the reference's) on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "block-row updates/s per sweep (fp64)"
UNIT = "block-rows/s"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._th = threading.Thread(target=run, daemon=True)
        self._th.start()

    def stop(self):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for k, nm in enumerate(names):
                if len(s) > 3 + k and s[3 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def sweep_bytes(n, e, b, lanes=1):
    """Algorithmic bytes of one (batched) complex harmonic sweep, stored-factor ILU
    (SURVEY.md 8(d)): the real A5 of the matvec (N+2E) b^2 8 once, and per lane 2E b^2 16
    (L,U) + N (b^2 16 + 4b) (pivot LU + piv) + N 8 (shift) + 5 N b 16 (rhs, x r/w, r, z)."""
    per_lane = 2 * e * b * b * 16 + n * (b * b * 16 + 4 * b) + n * 8 + 5 * n * b * 16
    return (n + 2 * e) * b * b * 8 + lanes * per_lane


def rb_sweep_bytes(n, n0, e, b, lanes=1):
    """Algorithmic bytes of one batched complex harmonic sweep on the 2-colour path (rb.cuh)
    over `lanes` harmonics, every array counted once: the shared real A5 (N+2E) b^2 8 once,
    and per lane: shift N 8, rhs N b 16, x r/w 2 N b 16, z (colour 1) r/w 2 N1 b 16,
    r (colour 0) r/w 2 N0 b 16, pivot LU + piv N (b^2 16 + 4 b), inv(U_kk) of colour 0
    N0 b^2 16."""
    n1 = n - n0
    per_lane = (n * 8 + n * b * 16 + 2 * n * b * 16 + 2 * n1 * b * 16 + 2 * n0 * b * 16
                + n * (b * b * 16 + 4 * b) + n0 * b * b * 16)
    return (n + 2 * e) * b * b * 8 + lanes * per_lane


def cpu_baseline(config, scale, seconds_hint=20.0):
    """The CPU path on the host cores: the oracle restatement (generic LA bitwise the
    reference's) running full pseudo-steps of the same configuration at a reduced size."""
    from oracle.oracle import Oracle
    from paper_2404_01407_b200.cases import make_case

    c = make_case(config, scale=scale)
    workers = max(1, min(len(c.omegas), os.cpu_count() or 1))  # the reference's harmonic workers
    orc = Oracle(workers=workers)
    s = orc.solver(c.mesh, c.mesh.pattern(), c.scheme, c.omegas, c.forcing, c.mean0)
    rows = 0
    t0 = time.perf_counter()
    steps = 0
    while True:
        s.outer_iteration()
        steps += 1
        if time.perf_counter() - t0 > seconds_hint or steps >= 3:
            break
    dt = time.perf_counter() - t0
    rows = sum(r[0] for r in s.reports()) * c.mesh.n
    return {"value": rows / dt, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": f"{steps} pseudo-step(s) of {config} at scale {scale} ({c.mesh.n} nodes, "
                      f"{len(c.omegas)} harmonics), oracle/fnlh_oracle.c, {workers} harmonic worker thread(s) "
                      f"(host has {os.cpu_count()}), {dt:.1f} s"}


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2404_01407_b200.cases import make_case
    from oracle.oracle import Oracle

    scale = args.ref_scale
    c = make_case(args.config, scale=scale)
    workers = max(1, min(len(c.omegas), os.cpu_count() or 1))  # all the threads the reference's scheme uses
    orc = Oracle(workers=workers)
    s = orc.solver(c.mesh, c.mesh.pattern(), c.scheme, c.omegas, c.forcing, c.mean0)
    for _ in range(args.warmup):
        s.outer_iteration()
    r0 = sum(r[0] for r in s.reports())
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s.outer_iteration()
    dt = time.perf_counter() - t0
    rows = (sum(r[0] for r in s.reports()) - r0) * c.mesh.n
    v = rows / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": {"workload": f"{args.config} pseudo-step, CPU sample at scale {scale} ({c.mesh.n} nodes)",
                       "harmonics": len(c.omegas), "l2": "inputs resident in host memory"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port",
                             "sample": f"{args.steps} pseudo-steps of {args.config} at scale {scale} "
                                       f"({c.mesh.n} nodes), oracle/fnlh_oracle.c, {workers} harmonic worker "
                                       f"thread(s) (host has {os.cpu_count()})"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--ref-scale", type=float, default=0.4)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sweeps", type=int, default=10, help="sweeps in the roofline leg")
    ap.add_argument("--mode", default="replicas", choices=["replicas", "shard"],
                    help="N>1: independent C2 replicas per rank (weak scaling) or one C2 instance with its "
                         "harmonics sharded over the ranks, fields exchanged by NCCL broadcast (strong scaling)")
    ap.add_argument("--workers", type=int, default=0,
                    help="harmonic lanes (SchemeConfig::workers); 0 = one per harmonic (<= 8)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)

    rank, world, local = dist_env()
    import torch

    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        dist = None
    os.environ.setdefault("CUDA_VISIBLE_DEVICES_LOCAL", str(local))
    from paper_2404_01407_b200._lib import check, lib, require_gpu
    from paper_2404_01407_b200.cases import make_case
    from paper_2404_01407_b200.solver import FnlhSolver

    require_gpu()
    check(lib().fnlh_set_device(local))  # this rank's GPU for the library's own runtime calls
    c = make_case(args.config, scale=args.scale)
    if args.workers != 1:
        c = make_case(args.config, scale=args.scale, workers=args.workers or min(len(c.omegas), 8))
    m = c.mesh
    pat = m.pattern()
    n, b = m.n, m.b
    E = (len(pat["col_idx"]) - n) // 2
    s = FnlhSolver(m, c.scheme, c.omegas, c.forcing, c.mean0, pattern=pat)
    shard = args.mode == "shard" and world > 1
    if shard:
        from paper_2404_01407_b200.shard import HarmonicShards
        stepper = HarmonicShards(s, len(c.omegas), n * b, device=f"cuda:{local}")
    else:
        stepper = s

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        stepper.outer_iteration()
    barrier()
    cnt0 = s.counters()
    nrep0 = len(s.reports()) if shard else 0
    launches0 = lib().fnlh_launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    dev_ms = 0.0
    phase = dict(lhs=0.0, harmonics=0.0, df=0.0, mean=0.0)
    for _ in range(args.steps):
        e = stepper.outer_iteration()
        cn = s.counters()
        dev_ms += cn["last_ms"]
        for k in phase:
            phase[k] += cn["phase_ms"][k] / args.steps
    barrier()
    clk = clocks.stop()
    launches = int(lib().fnlh_launch_count() - launches0)
    cnt1 = s.counters()
    rows = cnt1["row_updates"] - cnt0["row_updates"]
    if shard:  # the job's work once: every system's sweeps (identical report list on all ranks) on rank 0
        rows = sum(r[0] for r in s.reports()[nrep0:]) * n if rank == 0 else 0
    sweeps = cnt1["sweeps"] - cnt0["sweeps"]
    t = torch.tensor([dev_ms, float(rows)], dtype=torch.float64, device="cuda")
    if dist:
        tmax = t.clone()
        dist.all_reduce(tmax[0:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:2], op=dist.ReduceOp.SUM)
        t = torch.stack([tmax[0], t[1]])
    dev_ms_max, rows_all = float(t[0]), float(t[1])
    value = rows_all / (dev_ms_max * 1e-3)

    # e2e through the C ABI with host buffers: upload state, one pseudo-step, download state;
    # the host buffers are pinned (page-locked), as an application staging its fields would
    mean_h = torch.empty(n * b, dtype=torch.float64, pin_memory=True).numpy()
    amps_h = torch.empty(max(len(c.omegas), 1) * n * b * 2, dtype=torch.float64,
                         pin_memory=True).numpy().view(np.complex128).reshape(max(len(c.omegas), 1), n * b)
    mean_h, amps_h = s.state(out=(mean_h, amps_h))
    h2d = mean_h.nbytes + amps_h.nbytes
    d2h = h2d
    cnt2 = s.counters()
    nrep2 = len(s.reports()) if shard else 0
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if shard:
            s.set_state(mean_h, amps_h)
            stepper.outer_iteration()
            mean_h, amps_h = s.state(out=(mean_h, amps_h))
        else:  # one call on host buffers, transfers overlapped with the step
            s.outer_iteration_host(mean_h, amps_h)
    barrier()
    e2e_s = time.perf_counter() - t0
    rows_e2e = s.counters()["row_updates"] - cnt2["row_updates"]
    if shard:
        rows_e2e = sum(r[0] for r in s.reports()[nrep2:]) * n if rank == 0 else 0
    te = torch.tensor([e2e_s, float(rows_e2e)], dtype=torch.float64, device="cuda")
    if dist:
        tm = te.clone()
        dist.all_reduce(tm[0:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(te[1:2], op=dist.ReduceOp.SUM)
        te = torch.stack([tm[0], te[1]])
    e2e_value = float(te[1]) / float(te[0])

    # roofline leg: the harmonic relaxation sweep as the product path runs it (all lanes)
    info = s.info()
    lanes = s.lanes()
    if lanes > 1:
        s.time_sweeps_batch(lanes, 2)
        sweep_ms = s.time_sweeps_batch(lanes, args.sweeps) / args.sweeps
    else:
        sweep_ms = s.time_sweeps(0, args.sweeps) / args.sweeps
    if info["red_black"]:
        bytes_sweep = rb_sweep_bytes(n, info["n0"], E, b, lanes)
        kname = (f"2-colour ILU(0)-Richardson sweep, reference operation order (k_rb_colour0 + k_rbx_colour1), "
                 f"{lanes} harmonic lane(s) per launch")
        formula = f"rb_sweep_bytes(lanes={lanes})"
    else:
        bytes_sweep = sweep_bytes(n, E, b, lanes)
        kname = f"level-scheduled ILU(0)-Richardson sweep (fwd/bwd levels + matvec), {lanes} harmonic lane(s)"
        formula = f"sweep_bytes(stored-factor, lanes={lanes})"
    peak, peak_kind = peaks()
    achieved = bytes_sweep / (sweep_ms * 1e-3) / 1e9
    single = None
    if lanes > 1 and info["red_black"]:  # the same sweep for one harmonic alone, for reference
        s.time_sweeps(0, 2)
        ms1 = s.time_sweeps(0, args.sweeps) / args.sweeps
        b1 = rb_sweep_bytes(n, info["n0"], E, b, 1)
        single = {"ms_per_launch": ms1, "bytes_per_launch": b1, "achieved": b1 / (ms1 * 1e-3) / 1e9,
                  "frac": b1 / (ms1 * 1e-3) / 1e9 / peak, "unit": "GB/s"}
    traffic = None
    try:  # dram read + write of the same kernels from the committed ncu --set full capture
        name = "r1_sweep_ncu_c2_lanes3.json" if lanes == 3 else "r1_sweep_ncu_c2.json"
        with open(os.path.join(ROOT, "profiles", name)) as f:
            prof = json.load(f)
        if info["red_black"] and args.config == "c2" and args.scale == 1.0 and prof.get("lanes", 1) == lanes:
            traffic = prof["traffic_bytes_per_sweep"]
    except Exception:
        pass

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, cases.py)",
            "config": {"workload": f"{args.config}: {c.description}", "nodes": n, "edges": E, "b": b,
                       "harmonics": len(c.omegas), "pseudo_step": "outer_iteration (FD J, ILU, RK x (N_h+1), DF)",
                       "l2": f"inputs larger than L2 (LHS {s.lhs_bytes() / 1e9:.2f} GB resident)",
                       "parallelism": (f"harmonics sharded over {world} ranks (NCCL broadcast of fields)" if shard
                                       else f"replicas x{world}" if world > 1 else "1 GPU"),
                       "sweeps_per_step": sweeps / args.steps, "lhs_bytes": s.lhs_bytes(),
                       "workers": c.scheme.get("workers", 1), "harmonic_lanes": lanes,
                       "step_split_ms": {k: round(v, 3) for k, v in phase.items()}},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "kernel": kname, "bytes_formula": formula,
                         "bytes_per_launch": bytes_sweep, "ms_per_launch": sweep_ms, "peak_kind": peak_kind,
                         "sweep_rows_per_s": lanes * n / (sweep_ms * 1e-3), "single_lane": single},
            "clocks": clk, "gpu_launches": launches}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config, args.ref_scale)
        except Exception as ex:  # the baseline is informative; never fail the bench on it
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
