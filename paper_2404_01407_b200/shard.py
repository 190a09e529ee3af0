"""Harmonic sharding of the FNLH outer iteration across ranks.

One process per GPU.  Within an outer iteration every harmonic's RK step reads only the
frozen mean, the shared A5 and its own field (driver.cpp:193-244), so harmonic h is
relaxed on rank h % world.  Each rank holds a replica of the mesh, A5, the mean ILU and
its own complex ILU workspace(s) (LHS bytes per rank independent of N_h).  The only
exchange is the harmonic fields themselves, once per outer iteration, before the
deterministic flux: one broadcast per harmonic from its owner over NCCL (NVLink /
NVSwitch).  DF's nq quadrature residuals are then shared out in consecutive blocks of
points and their sum is chained rank to rank in k order (one N b vector per hop, then one
broadcast), and the mean step runs redundantly on every rank, so every rank holds bitwise
the same state as a single-GPU run (no reduction changes any summation order; partial
sums are never all-reduced).

The reference runs the same decomposition on host threads (`workers`,
driver.cpp:246-265): every harmonic runs, successful ones are committed, and the first
error by harmonic index is rethrown.  Here every owner's field is broadcast even when a
rank failed, and the error of the lowest failing harmonic (FnlhError, original code) is
raised on every rank after the exchange, so all ranks leave the iteration in the same
state.

`solver` is anything with phase_harmonics / harmonic_reports / phase_mean and either
copy_amps (device solver: FnlhSolver, fields staged through a torch CUDA buffer) or
get_amps / put_amps (host fields, e.g. a CPU stand-in under the gloo backend in tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def owner(h: int, world: int) -> int:
    """Rank that relaxes harmonic h (round robin, driver.cpp:250 `hi += nthreads`)."""
    return h % world


class HarmonicShards:
    def __init__(self, solver, nh: int, field_len: int, group=None, device=None, split_df=True):
        self.s = solver
        self.split_df = split_df and hasattr(solver, "df_terms")
        self.nh = nh
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.owned = [1 if owner(h, self.world) == self.rank else 0 for h in range(nh)]
        self.device = device
        self.field_len = field_len  # complex entries per harmonic field (N * b)
        self._buf = None
        self.tdev = torch.device(device or "cuda") if hasattr(solver, "copy_amps") else torch.device("cpu")
        if hasattr(solver, "copy_amps"):
            self._buf = torch.empty(2 * field_len, dtype=torch.float64, device=self.tdev)
        self._terms = self._acc = None

    def _exchange_field(self, h: int):
        src = owner(h, self.world)
        if self._buf is not None:  # device fields: stage through one buffer, NCCL broadcast
            if self.rank == src:
                self.s.copy_amps(h, self._buf.data_ptr(), True)  # returns once _buf holds the field
            dist.broadcast(self._buf, src=src, group=self.group)
            # dist.broadcast only orders torch's current stream after the collective; the
            # library copies on its own stream, so wait here: the receiver must not read _buf
            # before the data lands, the sender must not overwrite it (next harmonic) while
            # NCCL still reads it
            torch.cuda.current_stream(self._buf.device).synchronize()
            if self.rank != src:
                self.s.copy_amps(h, self._buf.data_ptr(), False)
        else:
            t = torch.from_numpy(self.s.get_amps(h).view("float64").copy()) if self.rank == src else \
                torch.empty(2 * self.field_len, dtype=torch.float64)
            dist.broadcast(t, src=src, group=self.group)
            if self.rank != src:
                self.s.put_amps(h, t.numpy().view("complex128"))

    def outer_iteration(self):
        """phase_harmonics on the owned harmonics, exchange, phase_mean.  Errors follow the
        reference's workers (driver.cpp:246-265): every harmonic runs, the owner's field of
        every harmonic (committed or, on the sequential path, left untouched) is broadcast so
        all ranks stay identical, and every rank raises the error of the lowest failing
        harmonic index with its original code / node / stage."""
        err = None
        h_norm = None
        try:
            h_norm = self.s.phase_harmonics(self.owned)
        except Exception as ex:  # captured, agreed on below (driver.cpp:248-264)
            fh = self.s.failed_harmonic() if hasattr(self.s, "failed_harmonic") else -1
            err = (fh, getattr(ex, "code", 7), str(ex), getattr(ex, "node", -1), getattr(ex, "stage", -1),
                   type(ex).__name__)
        mine = {h: (float(h_norm[h]), self.s.harmonic_reports(h)) for h in range(self.nh)
                if self.owned[h]} if err is None else {}
        gathered = [None] * self.world
        dist.all_gather_object(gathered, (err, mine), group=self.group)
        for h in range(self.nh):  # every field current on every rank, failing ranks included
            self._exchange_field(h)
        errors = [e for e, _ in gathered if e is not None]
        if errors:  # errors before the harmonics (-1) are the same on every rank and come first
            fh, code, msg, node, stage, kind = min(errors, key=lambda e: e[0])
            from ._lib import FnlhError
            e = FnlhError(code, f"harmonic shard (harmonic {fh}): {msg}", node, stage)
            e.harmonic = fh
            raise e
        norms, reports = [0.0] * self.nh, [[] for _ in range(self.nh)]
        for _, m in gathered:
            for h, (nv, reps) in m.items():
                norms[h], reports[h] = nv, reps
        if self.split_df and self.world > 1:
            self._deterministic_flux()
        return self.s.phase_mean(norms, reports)

    def _sync(self):
        if self.tdev.type == "cuda":
            torch.cuda.current_stream(self.tdev).synchronize()

    def _deterministic_flux(self):
        """DF with its nq quadrature residuals shared out: rank r evaluates the consecutive
        points [r K, (r+1) K) (fnlh_solver_df_terms), then the in-order sum is chained rank
        to rank -- receive the running sum, add the own terms in k order, pass it on -- so it
        is the reference's sequential sum (residual_ops.cpp:145-152) bit for bit; the last
        rank broadcasts it and every rank finishes DF = acc / nq - R(mean) in phase_mean."""
        nq = self.s.df_points()
        K = -(-nq // self.world)
        k0, k1 = min(nq, self.rank * K), min(nq, (self.rank + 1) * K)
        L = self.field_len
        if self._acc is None:
            self._acc = torch.zeros(L, dtype=torch.float64, device=self.tdev)
            self._terms = torch.empty(max(K, 1) * L, dtype=torch.float64, device=self.tdev)
        err = None
        try:
            if k1 > k0:
                self.s.df_terms(k0, k1, self._terms.data_ptr())
        except Exception as ex:  # the lowest rank's error is the reference's first (lowest k)
            err = (getattr(ex, "code", 7), str(ex), getattr(ex, "node", -1), getattr(ex, "stage", -1))
        errs = [None] * self.world
        dist.all_gather_object(errs, err, group=self.group)
        bad = [e for e in errs if e is not None]
        if bad:
            from ._lib import FnlhError
            code, msg, node, stage = bad[0]
            raise FnlhError(code, f"deterministic_flux (sharded): {msg}", node, stage)
        src = lambda r: dist.get_global_rank(self.group, r) if self.group is not None else r  # noqa: E731
        # NCCL moves the device vector directly; gloo (tests) only does point to point on host tensors
        wire = self._acc.cpu() if (self.tdev.type == "cuda" and dist.get_backend(self.group) == "gloo") else self._acc
        if self.rank > 0:
            dist.recv(wire, src=src(self.rank - 1), group=self.group)
            if wire is not self._acc:
                self._acc.copy_(wire)
            self._sync()
        if k1 > k0:
            self.s.df_accumulate(self._terms.data_ptr(), k1 - k0, self._acc.data_ptr(), k0 == 0)
        if wire is not self._acc:
            wire.copy_(self._acc)
        if self.rank < self.world - 1:
            dist.send(wire, dst=src(self.rank + 1), group=self.group)
            self._sync()
        dist.broadcast(wire, src=src(self.world - 1), group=self.group)
        if wire is not self._acc:
            self._acc.copy_(wire)
        self._sync()
        self.s.set_external_df(self._acc.data_ptr())
