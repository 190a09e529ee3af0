"""Boundary-state pow.  The device restates glibc's pow bit for bit (csrc/libm_pow.cuh, the
reference's libm); the correctly rounded fallback (oracle/cr_pow.h, csrc/cr_pow.cuh) is checked
against 60-digit decimal arithmetic, and its history-level gap to the reference is measured."""
import ctypes as C
import math
from decimal import Decimal, getcontext

import numpy as np


def test_cr_pow_correctly_rounded_and_glibc_gap(orc):
    lib = orc.lib
    lib.or_cr_pow.restype = C.c_double
    getcontext().prec = 60
    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.uniform(0.5, 2.0, 300), rng.uniform(0.99, 1.01, 300)])
    bad_cr = bad_glibc = 0
    for y in (3.5, 1.0 / 1.4):
        for x in xs:
            x = float(x)
            exact = (Decimal(x).ln() * Decimal(y)).exp()
            truth = float(exact)  # correctly rounded
            bad_cr += lib.or_cr_pow(C.c_double(x), C.c_double(y)) != truth
            bad_glibc += math.pow(x, y) != truth  # glibc pow, as the reference
    assert bad_cr == 0
    assert bad_glibc < 0.01 * 2 * len(xs)


def test_device_pow_is_glibc_bitwise():
    """The device's boundary-state pow (csrc/libm_pow.cuh) restates glibc's pow with the
    tables of the libm this process loaded: bitwise equal to math.pow (the reference's libm)
    on the boundary-state exponents and a wide log-uniform sweep, including arguments
    glibc misrounds (where the correctly rounded pow differs)."""
    from paper_2404_01407_b200._lib import lib, pow_mode
    L = lib()
    assert pow_mode() == "glibc", L.fnlh_pow_mode_info().decode()
    rng = np.random.default_rng(11)
    xs = np.concatenate([rng.uniform(0.8, 1.2, 20000), np.exp2(rng.uniform(-40, 40, 5000))])
    misrounded = 0
    for y in (3.5, 1.0 / 1.4, -2.25):
        for x in xs:
            x = float(x)
            g = math.pow(x, y)
            assert L.fnlh_pow(x, y) == g, (x, y)
    getcontext().prec = 60
    for x in xs[:20000]:
        x = float(x)
        for y in (3.5, 1.0 / 1.4):
            misrounded += math.pow(x, y) != float((Decimal(x).ln() * Decimal(y)).exp())
    assert misrounded > 0  # the cases a correctly rounded pow would get "wrong" vs the reference


def test_pow_rounding_matters_for_history(ref):
    """Why the device needs glibc's rounding: on the reference's own nozzle, 20 pseudo-steps
    of the restatement with a correctly rounded boundary pow drift from the reference by
    more than the north_star history bar (1e-8), while glibc's rounding reproduces it."""
    from oracle.oracle import Oracle
    from helpers import NOZZLE_CASE, embed, forcing_triplets, line_mesh_from_ref
    drift = {}
    for mode in ("glibc", "cr"):
        rs = ref.solver(NOZZLE_CASE.format(nx=64, nh=2))
        noz = rs.noz
        m = line_mesh_from_ref(noz)
        forc = np.stack([forcing_triplets(f) for f in noz.forcing])
        o = Oracle(pow_mode=mode).solver(m, noz.pattern(5), dict(implicit=1), noz.omega, forc,
                                         embed(noz.initial_mean(), noz.n))
        s = np.sqrt(5 / 3)
        d = 0.0
        for _ in range(20):
            er, eo = rs.outer_iteration(), o.outer_iteration()
            d = max(d, abs(eo["rz"] * s / er["rz"] - 1), abs(eo["resid_mean"] * s / er["resid_mean"] - 1))
        drift[mode] = d
    assert drift["glibc"] < 1e-14
    assert drift["cr"] > 1e-8
