#!/usr/bin/env python
"""Benchmark of the FNLH implicit pseudo-time hot path on B200.

Workload: BASELINE.json configs[3] (C4), the largest configuration that fits one GPU:
hex sector 256x128x128, 4,276,737 nodes, 5 conservative variables, 10 harmonics,
implicit scheme (tol 1e-2, <= 10 sweeps), harmonics in 8 lanes (SchemeConfig::workers).
A step is one pseudo-step (FnlhSolver::outer_iteration, driver.cpp:157-333): FD
Jacobian, A5 + real ILU(0), per harmonic complex ILU(0) + RK(5,3) with the
linearized residual and ILU-Richardson sweeps, DF, mean RK(5,3).  --config c2 runs C2.

  value = block-row updates performed in the timed steps (sum over every stage solve
          of iterations x N) / device time of the timed steps, all ranks
  e2e   = same through the C ABI with host buffers (state uploaded and downloaded
          every step)
  roofline = the harmonic relaxation sweep (smoothed_solve iteration) as the product
          runs it (all lanes in one batched launch pair), algorithmic bytes
          (rb_sweep_bytes) / CUDA-event time of the batched sweep

--impl reference: the reference's own CPU implementation on the same full-size C4
harmonic systems (oracle/_ref: the unmodified reference compiled from its sources):
its Ilu<complex>::factorize and smoothed_solve sweeps on min(N_h, cores, memory)
concurrent harmonic workers (driver.cpp:246-265), rank 0 only; the mesh, pattern and
FD Jacobian are built on the host (the restatement), so no product code is loaded.

Multi-GPU (--gpus N under torchrun): --mode shard (default for N > 1) relaxes the
harmonics of one C4 instance on their owner ranks (h % N) with the fields exchanged by
NCCL broadcast, "scaling": "strong"; --mode replicas runs one instance per rank.
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


ALPHA5 = 1.0  # rk.hpp:27, alpha of stage 5 (the operator every stage solve uses)


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count() or 1


def ref_worker_count(n_h, per_worker_bytes, reserve=16e9):
    """The reference's harmonic workers that fit: min(N_h, host cores, host memory)."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64e9
    return max(1, min(n_h, os.cpu_count() or 1, int((avail - reserve) // per_worker_bytes)))


class RefHarmonicWorkers:
    """Full-size harmonic systems on the reference's own objects (oracle/_ref, the unmodified
    reference): A5 = build_lhs_mean(J) (rk.cpp:5-30) shared read-only, and per worker the
    complex workspace shift_diagonal(A5, i omega V / (Gamma alpha_5)) (build_lhs_harmonic,
    rk.cpp:32-39), Ilu<complex>::factorize (sparse.cpp:187-257) and smoothed_solve sweeps
    (sparse.hpp:295-331) -- what one harmonic worker of driver.cpp:246-265 holds."""

    def __init__(self, case, pat, J, n_workers):
        import threading
        from oracle.oracle import RefLib
        self.ref = RefLib()
        sch = case.scheme
        sigma = sch["sigma_cfl"] if sch["sigma_cfl"] > 0 else 50.0  # driver.hpp:33-41 implicit default
        A5 = self.ref.build_lhs_mean(pat, J, 1, sigma, sch["eps_relax"], 5)
        self.lhs = self.ref.lhs_create(pat, A5)
        del A5
        n, b = case.mesh.n, case.mesh.b
        ga5 = (1.0 / sch["eps_relax"]) * ALPHA5
        rng = np.random.default_rng(4242)
        self.workers = [None] * n_workers
        self.factor_s = [0.0] * n_workers
        self.n = n

        def make(t):
            shift = case.omegas[t] * case.mesh.vol / ga5
            rhs = rng_rhs[t]
            self.workers[t], self.factor_s[t] = self.ref.hworker_create(self.lhs, shift, rhs)

        rng_rhs = [rng.standard_normal(n * b) + 1j * rng.standard_normal(n * b) for _ in range(n_workers)]
        th = [threading.Thread(target=make, args=(t,)) for t in range(n_workers)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if any(w is None for w in self.workers):
            raise RuntimeError("reference harmonic worker setup failed")

    def sweep_all(self, count=None):
        """One smoothed_solve iteration on each of the first `count` workers concurrently
        (ctypes releases the GIL): wall seconds."""
        import threading
        ws = self.workers[: count or len(self.workers)]
        th = [threading.Thread(target=self.ref.hworker_sweeps, args=(w, 1)) for w in ws]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        return time.perf_counter() - t0

    def close(self):
        for w in self.workers:
            if w:
                self.ref.hworker_destroy(w)
        self.ref.lhs_destroy(self.lhs)


def per_worker_bytes(n, nnzb, b):
    """Host bytes of one reference harmonic worker: complex workspace + Ilu<complex> (vals,
    diag_lu, diag_inv, pivots) + the smoothed_solve vectors."""
    return nnzb * b * b * 16 * 2 + n * b * b * 16 * 2 + n * b * 4 + 6 * n * b * 16


def cpu_baseline(case, pat, J):
    """The reference's own CPU path (oracle/_ref) on a bounded sample of the same workload:
    the full-size harmonic systems of this configuration, one Richardson sweep each, with
    1 worker (1 core) and with min(N_h, cores, memory) concurrent workers."""
    model, cores = host_info()
    n, b = case.mesh.n, case.mesh.b
    W = ref_worker_count(len(case.omegas), per_worker_bytes(n, len(pat["col_idx"]), b))
    t0 = time.perf_counter()
    rw = RefHarmonicWorkers(case, pat, J, W)
    setup = time.perf_counter() - t0
    t1 = rw.sweep_all(1)
    tw = rw.sweep_all(W)
    rw.close()
    return {"value": W * n / tw, "unit": UNIT, "cores": W, "kind": "reference",
            "one_core": {"value": n / t1, "unit": UNIT, "seconds_per_sweep": t1},
            "workers": W, "seconds_per_sweep": tw, "host": {"cpu_model": model, "nproc": cores},
            "factorize_seconds_per_worker": round(max(rw.factor_s), 2),
            "sample": f"one smoothed_solve sweep of each of {W} full-size {case.name} harmonic system(s) "
                      f"({n} nodes, nnzb {len(pat['col_idx'])}) on the reference's Ilu<complex> / smoothed_solve "
                      f"(oracle/_ref), {W} concurrent worker thread(s) on {cores} host cores ({model}); the 1-core "
                      f"number is one worker alone; setup (shift_diagonal + factorize, not timed) {setup:.0f} s"}


def reference_arm(args):
    """The reference's CPU implementation of the path, on the same full-size workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.oracle import Oracle
    from paper_2404_01407_b200.cases import make_case

    t0 = time.perf_counter()
    ov = {"order": args.order} if args.order else {}
    c = make_case(args.config, scale=args.scale, device=False, **ov)  # host restatement: no product code loaded
    pat = c.mesh.pattern(device=False)
    J, _ = Oracle().fd_jacobian(c.mesh, pat, c.mean0)  # the restatement (bitwise the device's, tests)
    n, b = c.mesh.n, c.mesh.b
    W = ref_worker_count(len(c.omegas), per_worker_bytes(n, len(pat["col_idx"]), b))
    rw = RefHarmonicWorkers(c, pat, J, W)
    del J
    setup = time.perf_counter() - t0
    for _ in range(args.warmup):
        rw.sweep_all()
    wall = 0.0
    for _ in range(args.steps):
        wall += rw.sweep_all()
    rw.close()
    v = W * n * args.steps / wall
    model, cores = host_info()
    loaded = [ln.split()[-1] for ln in open("/proc/self/maps") if "libfnlh_b200" in ln]
    E = (len(pat["col_idx"]) - n) // 2
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, cases.py)",
            "config": workload_config(c, n, E, b),
            "step": f"one smoothed_solve sweep (Ilu<complex>::apply + Bsr::matvec + norm, sparse.hpp:315-329) of "
                    f"each of {W} full-size harmonic systems, one reference harmonic worker thread each",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": W, "kind": "reference",
                             "host": {"cpu_model": model, "nproc": cores},
                             "sample": f"{args.steps} timed steps x {W} concurrent full-size {args.config} harmonic "
                                       f"sweeps on oracle/_ref (the unmodified reference), {cores} host cores "
                                       f"({model}); setup (host mesh, FD Jacobian, shift_diagonal, factorize) "
                                       f"{setup:.0f} s untimed"},
            "product_library_loaded": bool(loaded),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(c, n, E, b):
    """The workload keys, identical on both arms (same_config); run details go to "details"."""
    a5 = (n + 2 * E) * b * b * 8
    return {"workload": f"{c.name}: {c.description}", "nodes": n, "edges": E, "b": b, "harmonics": len(c.omegas),
            "l2": f"inputs larger than L2 (the shared LHS A5 alone is {a5 / 1e9:.2f} GB)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--order", default=None, choices=["rcm", "morton", "lex", "lexk"],
                    help="node numbering inside each colour (default: the configuration's)")
    ap.add_argument("--sweeps", type=int, default=10, help="sweeps in the roofline leg")
    ap.add_argument("--mode", default="shard", choices=["replicas", "shard"],
                    help="N>1: one instance with its harmonics sharded over the ranks, fields exchanged by NCCL "
                         "broadcast (strong scaling, default), or independent replicas per rank (weak scaling)")
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
    ov = {"order": args.order} if args.order else {}
    c = make_case(args.config, scale=args.scale, **ov)
    if args.workers != 1:
        c = make_case(args.config, scale=args.scale, workers=args.workers or min(len(c.omegas), 8), **ov)
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
    traffic, traffic_src = None, None
    try:  # dram read + write of the same kernels from the committed ncu --set full capture
        name = {("c4", 8): "r2_sweep_ncu_c4_lanes8.json", ("c2", 3): "r1_sweep_ncu_c2_lanes3.json",
                ("c2", 1): "r1_sweep_ncu_c2.json"}.get((args.config, lanes))
        if name and info["red_black"] and args.scale == 1.0:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                prof = json.load(f)
            if prof.get("lanes", 1) == lanes:
                traffic, traffic_src = prof["traffic_bytes_per_sweep"], f"profiles/{name}"
    except Exception:
        pass

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, cases.py)",
            "config": workload_config(c, n, E, b),
            "details": {
                       "pseudo_step": "outer_iteration (FD J, ILU, RK x (N_h+1), DF)",
                       "resident": f"LHS {s.lhs_bytes() / 1e9:.2f} GB in HBM",
                       "parallelism": (f"harmonics sharded over {world} ranks (NCCL broadcast of fields)" if shard
                                       else f"replicas x{world}" if world > 1 else "1 GPU"),
                       "sweeps_per_step": sweeps / args.steps, "lhs_bytes": s.lhs_bytes(),
                       "workers": c.scheme.get("workers", 1), "harmonic_lanes": lanes,
                       "step_split_ms": {k: round(v, 3) for k, v in phase.items()}},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": traffic_src, "kernel": kname, "bytes_formula": formula,
                         "bytes_per_launch": bytes_sweep, "ms_per_launch": sweep_ms, "peak_kind": peak_kind,
                         "sweep_rows_per_s": lanes * n / (sweep_ms * 1e-3), "single_lane": single},
            "clocks": clk, "gpu_launches": launches}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:  # the reference's CPU sweep on the same full-size systems; J from the device (bitwise the host's)
            del mean_h, amps_h
            from paper_2404_01407_b200.solver import Discretization
            J, _ = Discretization(m, pat).fd_jacobian(c.mean0)
            line["cpu_baseline"] = cpu_baseline(c, pat, J)
            del J
        except Exception as ex:  # the baseline is informative; never fail the bench on it
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
