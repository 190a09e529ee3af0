"""GPU: the device path against golden vectors written by the reference itself
(tests/golden/make_golden.py), so the B200 run pins against the reference even
where /root/reference is absent."""
import os

import numpy as np
import pytest

from paper_2404_01407_b200._lib import pow_mode
from helpers import embed, extract, extract_blocks, forcing_triplets, line_mesh_from_ref, nozzle_from_golden, rel

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("key", ["b5_z", "b5_d", "b3_z"])
@pytest.mark.parametrize("rb", [True, False])
def test_la_golden(key, rb):
    from paper_2404_01407_b200 import la
    from paper_2404_01407_b200.mesh import structured_sector
    g = np.load(os.path.join(GOLD, "la_hex4x3x3.npz"))
    b = int(key[1])
    cplx = key.endswith("z")
    pat = structured_sector(4, 3, 3, seed=11).pattern(b)
    P = la.Pattern.from_dict(pat)
    A = g[f"{key}_A"]
    shift = g[f"{key}_shift"] if cplx else None
    la.set_red_black(rb)
    try:
        f = la.ilu_factorize(P, A, shift)
        for k in ("vals", "diag_lu", "diag_piv", "diag_inv"):
            assert np.array_equal(f[k], g[f"{key}_{k}"]), k
        x, rep = la.smoothed_solve(P, A, g[f"{key}_rhs"], 1e-6, 6, shift)
        assert np.array_equal(x, g[f"{key}_x"])
        assert rep[0] == int(g[f"{key}_rep"][0])
    finally:
        la.set_red_black(True)


def test_nozzle_golden():
    from paper_2404_01407_b200.solver import Discretization, FnlhSolver
    noz = nozzle_from_golden(os.path.join(GOLD, "nozzle_nx64_h2.npz"))
    m = line_mesh_from_ref(noz)
    d = Discretization(m, noz.pattern(5))
    W5 = embed(noz.W3, noz.n)
    gi, _ = d.residual(W5, 1)
    assert np.array_equal(extract(gi, noz.n), noz.res1)
    gi2, _ = d.residual(W5, 2)
    assert np.array_equal(extract(gi2, noz.n), noz.res2)
    J5, _ = d.fd_jacobian(W5)
    assert pow_mode() == "glibc", "device pow is not the reference's libm rounding"
    assert np.array_equal(extract_blocks(J5, noz.nnzb), noz.J)
    li, _ = d.linearized_residual(W5, embed(noz.what3, noz.n, np.complex128), noz.omega[0],
                                  forcing_triplets(noz.forcing[0]))
    assert np.array_equal(extract(li, noz.n), noz.linres)
    forc = np.stack([forcing_triplets(f) for f in noz.forcing])
    s = FnlhSolver(m, dict(implicit=1), noz.omega, forc, embed(noz.mean0, noz.n), pattern=noz.pattern(5))
    k = np.sqrt(5 / 3)
    for it in range(20):  # the north_star bar is 1e-8; the device meets it to rounding of the RMS
        e = s.outer_iteration()
        assert abs(e["resid_mean"] * k / noz.hist[it, 1] - 1) < 1e-12, (it, e)
        assert abs(e["rz"] * k / noz.hist[it, 2] - 1) < 1e-12, (it, e)
    mean, amps = s.state()
    assert rel(extract(mean, noz.n), noz.mean20) < 1e-12
    assert rel(np.stack([extract(a, noz.n) for a in amps]), noz.amps20) < 1e-12
