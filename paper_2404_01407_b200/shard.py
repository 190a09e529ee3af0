"""Harmonic sharding of the FNLH outer iteration across ranks.

One process per GPU.  Within an outer iteration every harmonic's RK step reads only the
frozen mean, the shared A5 and its own field (driver.cpp:193-244), so harmonic h is
relaxed on rank h % world.  Each rank holds a replica of the mesh, A5, the mean ILU and
its own complex ILU workspace(s) (LHS bytes per rank independent of N_h).  The only
exchange is the harmonic fields themselves, once per outer iteration, before the
deterministic flux: one broadcast per harmonic from its owner over NCCL (NVLink /
NVSwitch).  DF and the mean step then run redundantly, in the same order, on every rank,
so every rank holds bitwise the same state as a single-GPU run (no reduction changes any
summation order; partial reconstructions are never all-reduced).

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
    def __init__(self, solver, nh: int, field_len: int, group=None, device=None):
        self.s = solver
        self.nh = nh
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.owned = [1 if owner(h, self.world) == self.rank else 0 for h in range(nh)]
        self.device = device
        self.field_len = field_len  # complex entries per harmonic field (N * b)
        self._buf = None
        if hasattr(solver, "copy_amps"):
            self._buf = torch.empty(2 * field_len, dtype=torch.float64, device=device or "cuda")

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
        return self.s.phase_mean(norms, reports)
