"""The five BASELINE.json configurations as seeded synthetic inputs.

None of them is a public benchmark: meshes, mean states, eddy-viscosity fields and
forcing amplitudes are generated here from documented seeds (numpy PCG64).  Flow is
nondimensional (rho = 1, c = 1, p = 1/gamma, R = 1/gamma so T = 1); inlet total
conditions are the isentropic totals of the nominal Mach number, the outlet static
pressure is the nominal p.  Mapping of BASELINE wording:
"N relaxation sweeps" = linear_max_iter N with linear_tol 1e-14; "coloured SGS" =
ILU(0)-Richardson in a colour-major ordering; "explicit 4-stage RK" = the
reference's explicit RK(5,3) on one grid.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .mesh import structured_sector

GAMMA = 1.4


@dataclasses.dataclass
class Case:
    name: str
    mesh: object
    scheme: dict
    omegas: np.ndarray
    forcing: np.ndarray       # [nh, 3*n_boundary] complex
    mean0: np.ndarray         # [n*b]
    pseudo_steps: int
    description: str


SPECS = {
    "c1": dict(cells=(32, 16, 8), geometry="channel", periodic_j=True, tets=False, b=5, mach=0.5, nh=1,
               sigma=10.0, max_iter=4, tol=1e-14, steps=20, seed=101,
               desc="hex channel 32x16x8, periodic pitch, M0.5 + 1% seeded perturbation, 1 harmonic, CFL 10, "
                    "20 pseudo-steps, 4 sweeps"),
    "c2": dict(cells=(128, 64, 48), geometry="annular", periodic_j=False, tets=False, b=5, mach=0.6, nh=3,
               sigma=-1.0, max_iter=10, tol=1e-2, steps=50, seed=202, swirl=True,
               desc="annular hex sector 128x64x48, r 0.5-1.0, 10 deg pitch, permuted+RCM, M0.6 + seeded radial "
                    "swirl, 3 harmonics, 50 pseudo-steps"),
    "c3": dict(cells=(160, 96, 64), geometry="annular", periodic_j=False, tets=True, jitter=0.05, b=5, mach=0.7,
               nh=5, sigma=-1.0, max_iter=8, tol=1e-14, steps=3, seed=303,
               desc="Kuhn 6-tet split of 160x96x64 hex sector, 5% jitter, M0.7, 5 harmonics, 8 sweeps"),
    "c4": dict(cells=(256, 128, 128), geometry="annular", periodic_j=False, tets=False, b=5, mach=0.6, nh=10,
               sigma=-1.0, max_iter=10, tol=1e-2, steps=2, seed=404,
               desc="hex sector 256x128x128, 10 harmonics (memory-scaling test)"),
    "c5": dict(cells=(160, 96, 64), geometry="annular", periodic_j=False, tets=True, jitter=0.05, b=6, mach=0.7,
               nh=5, sigma=-1.0, max_iter=8, tol=1e-14, steps=3, seed=505, mu_range=(1e-6, 1e-3),
               desc="C3 mesh, b=6 (Euler + SA-like scalar), seeded nu_t log-U[1e-6,1e-3], 5 harmonics"),
}


def make_case(name: str, scale: float = 1.0, nh: int | None = None, implicit: bool = True, permute: bool = True,
              workers: int = 1, device: bool | None = None, **overrides) -> Case:
    """Build config `name` ('c1'..'c5').  `scale` shrinks the cell counts (parity tests run
    the same configuration at sizes the CPU oracle finishes in seconds).  `device`: build the
    mesh with the library's kernels (None: when a GPU is present) or on the host (False, the
    bit-identical restatement: the CPU reference arm, which must not load the library)."""
    spec = dict(SPECS[name])
    spec.update(overrides)
    ci, cj, ck = spec["cells"]
    if scale != 1.0:
        ci, cj, ck = (max(4, int(round(c * scale))) for c in (ci, cj, ck))
        if spec["periodic_j"] and cj % 2:
            cj += 1
    rng = np.random.default_rng(spec["seed"])
    mach = spec["mach"]
    p = 1.0 / GAMMA
    R = 1.0 / GAMMA
    T = p / R
    fac = 1.0 + 0.5 * (GAMMA - 1.0) * mach * mach
    gas = dict(gamma=GAMMA, gas_constant=R, p0=p * fac ** (GAMMA / (GAMMA - 1.0)), T0=T * fac, p_out=p,
               forcing_scale=p)
    b = spec["b"]
    nt_in = 1e-3 if b == 6 else 0.0
    m = structured_sector(ci, cj, ck, geometry=spec["geometry"], periodic_j=spec["periodic_j"], tets=spec["tets"],
                          jitter=spec.get("jitter", 0.0), seed=spec["seed"], b=b, permute=permute, gas=gas,
                          nt_in=nt_in, mu_range=spec.get("mu_range"), device=device, order=spec.get("order", "rcm"),
                          colouring=spec.get("colouring", "structural"))
    n = m.n
    W = np.zeros((n, b))
    W[:, 0] = 1.0 * (1.0 + 0.01 * rng.uniform(-1, 1, n))
    W[:, 1] = mach * (1.0 + 0.01 * rng.uniform(-1, 1, n))
    W[:, 2] = 0.01 * mach * rng.uniform(-1, 1, n)
    W[:, 3] = 0.01 * mach * rng.uniform(-1, 1, n)
    W[:, 4] = p
    if spec.get("swirl"):
        X = m.coords
        r = np.sqrt(X[:, 1] ** 2 + X[:, 2] ** 2)
        th = np.arctan2(X[:, 2], X[:, 1])
        s = (r - r.min()) / max(r.max() - r.min(), 1e-12)
        a = rng.uniform(-0.1, 0.1, 3)
        vt = mach * sum(a[k] * np.sin((k + 1) * np.pi * s) for k in range(3))
        W[:, 2] += -vt * np.sin(th)
        W[:, 3] += vt * np.cos(th)
    if b == 6:
        W[:, 5] = nt_in * (1.0 + 0.01 * rng.uniform(-1, 1, n))
    nh_ = spec["nh"] if nh is None else nh
    omegas = 2.0 * np.pi * np.arange(1, nh_ + 1)
    nbf = m.n_boundary
    forcing = np.zeros((nh_, 3 * nbf), np.complex128)
    inlet = np.flatnonzero(m.fbc[m.fbc >= 0] == 0)
    for h in range(nh_):
        ph = rng.uniform(0, 2 * np.pi)
        forcing[h, 3 * inlet + 1] = 1e-3 * p * np.exp(1j * ph)
    scheme = dict(implicit=1 if implicit else 0, sigma_cfl=spec["sigma"] if implicit else -1.0, eps_relax=0.6,
                  linear_tol=spec["tol"], linear_max_iter=spec["max_iter"], target_drop_orders=8.0,
                  max_outer_iters=spec["steps"], workers=workers)
    return Case(name=name, mesh=m, scheme=scheme, omegas=omegas, forcing=forcing, mean0=W.reshape(-1),
                pseudo_steps=spec["steps"], description=spec["desc"])
