"""The device's boundary-state pow is correctly rounded (oracle/cr_pow.h is its C copy).
Checked against 60-digit decimal arithmetic; glibc's pow (the reference's libm) is
measured against the same truth so the residual oracle-vs-reference gap is explicit."""
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
