"""Time-accurate reference solver and harmonic extraction (SPEC `oracle_urans`).

The reference declares this module in oracle.hpp:28-52 (`unsteady_solve`,
`extract_harmonics`, `compare_amplitudes`, `TimeSeries`, `OracleOptions`) and ships no
implementation.  The time integration runs on the device through the C ABI
(`fnlh_solver_unsteady`, csrc/urans.cu): classical 4-stage explicit integration of
V dQ/dt = -R(W, t) with the FNLH residual itself (order 2), boundaries in perturbation mode
referenced to the steady state and forced with sum_l 2 Re(f_l e^{i omega_l t}), at a global
stable step, marched until the period-to-period relative L2 change is below
`periodic_tol`, then one period sampled uniformly.  The DFT extraction and the amplitude
comparison are small host reductions over the samples (numpy).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import FnlhError, check, lib, ptr, f64

_i, _d = C.c_int, C.c_double


@dataclass
class OracleOptions:  # oracle.hpp:21-27
    samples_per_period: int = 32  # raised to 4 l_max + 2 when too small
    cfl: float = 0.7
    periodic_tol: float = 1e-9    # period-to-period relative L2 change
    max_periods: int = 200
    min_periods: int = 2


@dataclass
class TimeSeries:  # oracle.hpp:14-19
    period: float                 # base period T of the forcing
    samples: np.ndarray           # [S, N*b] primitive states at t_k = k T / S over the final period
    info: dict = field(default_factory=dict)

    def sample_count(self) -> int:
        return int(self.samples.shape[0])


def base_frequency(omegas, rel_tol=1e-9):
    """HarmonicSpec::base_frequency / max_multiple (case.cpp:10-44) -> (base, l_max)."""
    ws = [float(w) for w in omegas if w > 0.0]
    if not ws:
        return 0.0, 0
    scale = max(ws)
    g = ws[0]
    for w in ws[1:]:
        a, b = max(g, w), min(g, w)
        while b > rel_tol * scale:
            a, b = b, math.fmod(a, b)
        g = a
    if g < 1e-6 * scale or any(abs(w / g - round(w / g)) > 1e-6 for w in ws):
        raise FnlhError(1, "harmonic frequencies are incommensurate")
    return g, max(int(round(w / g)) for w in ws)


def unsteady_solve(solver, steady=None, opt: OracleOptions | None = None) -> TimeSeries:
    """unsteady_solve(disc, steady, spec, opt) (oracle.hpp:28-33) for the mesh, frequencies
    and boundary forcing of `solver` (a FnlhSolver); `steady` defaults to its current mean.
    NonConvergenceError (status 8) when the period cap is hit first; the exception carries
    the last period's series as `.timeseries`."""
    opt = opt or OracleOptions()
    base, lmax = base_frequency(solver.omegas)
    if lmax == 0:
        raise FnlhError(1, "unsteady_solve: needs time-periodic forcing (a positive frequency)")
    S = max(opt.samples_per_period, 4 * lmax + 2)
    n = solver.m.n * solver.m.b
    out = np.zeros((S, n))
    info = np.zeros(5)
    st = lib().fnlh_solver_unsteady(solver.h, None if steady is None else ptr(f64(steady)),
                                    _i(opt.samples_per_period), _d(opt.cfl), _d(opt.periodic_tol),
                                    _i(opt.max_periods), _i(opt.min_periods), ptr(out), ptr(info))
    ts = TimeSeries(period=2.0 * math.pi / base, samples=out[: int(info[0]) or S],
                    info=dict(samples=int(info[0]), steps_per_period=int(info[1]), dt=float(info[2]),
                              periods=int(info[3]), last_change=float(info[4])))
    try:
        check(st)
    except FnlhError as ex:
        ex.timeseries = ts
        raise
    return ts


def extract_harmonics(ts: TimeSeries, omegas):
    """extract_harmonics (oracle.hpp:35-40): DFT over the sampled period under the
    conjugate-pair convention W(t) = mean + sum_l 2 Re(W_l e^{i omega_l t}), i.e.
    W_l = (1/S) sum_k W(t_k) e^{-i omega_l t_k}.  Frequencies must sit on the DFT grid
    (integer multiples of 2 pi / T below S/2); zero-frequency entries extract as zero."""
    S = ts.sample_count()
    w0 = 2.0 * math.pi / ts.period
    mean = ts.samples.mean(axis=0)
    amps = np.zeros((len(omegas), ts.samples.shape[1]), np.complex128)
    k = np.arange(S)
    for l, om in enumerate(omegas):
        if om == 0.0:
            continue
        m = om / w0
        if abs(m - round(m)) > 1e-6 or not (0 < round(m) < S / 2):
            raise FnlhError(1, f"extract_harmonics: frequency {om} is off the DFT grid of the series")
        ph = np.exp(-2j * math.pi * round(m) * k / S)
        amps[l] = ph @ ts.samples / S
    return mean, amps


def interior_mask(mesh, b, width=2):
    """Nodes more than `width` cells from either x-boundary (oracle.hpp:48-52)."""
    if mesh.ijk is None:
        raise FnlhError(1, "compare_amplitudes: the mesh has no structured x index")
    i = mesh.ijk[:, 0]
    keep = (i >= i.min() + width) & (i <= i.max() - width)
    return np.repeat(keep, b)


def compare_amplitudes(fnlh_amps, oracle_amps, mesh, width=2):
    """compare_amplitudes (oracle.hpp:47-52): per-harmonic relative L2 error over interior
    nodes -> [(index, rel_l2)]; ConfigError when the two sides differ in shape."""
    a = np.asarray(fnlh_amps, np.complex128)
    o = np.asarray(oracle_amps, np.complex128)
    if a.shape != o.shape:
        raise FnlhError(1, "compare_amplitudes: harmonic specs differ")
    keep = interior_mask(mesh, a.shape[1] // mesh.n, width)
    out = []
    for l in range(a.shape[0]):
        den = np.linalg.norm(o[l][keep])
        out.append((l, float(np.linalg.norm((a[l] - o[l])[keep]) / den) if den > 0 else 0.0))
    return out
