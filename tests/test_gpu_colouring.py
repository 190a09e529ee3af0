"""Greedy colouring on the device (fnlh_greedy_colour) for a mesh without structured
indices -- the C3 Kuhn tets with their node graph randomly permuted -- equals the host
restatement colour for colour; the colour-major RCM ordering it gives runs the
level-scheduled path with one ILU(0) level per colour, and the device ILU(0) factors, the
substitution and the Richardson iterates on that ordering are bitwise those of the reference
itself (oracle/_ref); two outer iterations match the restatement."""
import numpy as np
import pytest

from paper_2404_01407_b200.cases import make_case
from paper_2404_01407_b200.mesh import graph_csr, greedy_colouring

pytestmark = pytest.mark.gpu


def test_device_colouring_equals_host():
    for name, scale in (("c3", 0.15), ("c2", 0.1)):
        c = make_case(name, scale=scale, device=False)
        m = c.mesh
        inter = m.fbc < 0
        rp, ci = graph_csr(m.n, m.fa[inter], m.fb[inter])
        for seed in (1, 99):
            assert np.array_equal(greedy_colouring(m.n, rp, ci, seed, device=True),
                                  greedy_colouring(m.n, rp, ci, seed, device=False)), (name, seed)


def test_greedy_ordering_ilu_bitwise_vs_reference(ref, orc_dev):
    from paper_2404_01407_b200 import la
    from paper_2404_01407_b200.solver import FnlhSolver
    c = make_case("c3", scale=0.08, nh=2, colouring="greedy")
    m = c.mesh
    ncol = int(m.colour.max()) + 1
    pat = m.pattern()
    P = la.Pattern.from_dict(pat)
    assert P.levels() == (ncol, ncol)
    rng = np.random.default_rng(21)
    A = rng.standard_normal((len(pat["col_idx"]), 5, 5)) * 0.1
    A[pat["diag_idx"]] += 4 * np.eye(5)
    shift = rng.uniform(0.5, 2.0, m.n)
    Az = A.astype(np.complex128)
    Az[pat["diag_idx"]] += 1j * np.eye(5) * shift[:, None, None]
    fr = ref.ilu_factorize(pat, Az.reshape(-1))
    fd = la.ilu_factorize(P, A.reshape(-1), shift)
    for k in fr:
        assert np.array_equal(fd[k], fr[k]), k
    rhs = rng.standard_normal(m.n * 5) + 1j * rng.standard_normal(m.n * 5)
    xr, rr = ref.smoothed_solve(pat, Az.reshape(-1), rhs, 1e-3, 6)
    xd, rd = la.smoothed_solve(P, A.reshape(-1), rhs, 1e-3, 6, shift)
    assert np.array_equal(xd, xr) and rd[0] == rr[0]
    g = FnlhSolver(m, c.scheme, c.omegas, c.forcing, c.mean0)
    o = orc_dev.solver(m, pat, c.scheme, c.omegas, c.forcing, c.mean0)
    for _ in range(2):
        eg, eo = g.outer_iteration(), o.outer_iteration()
        assert abs(eg["resid_mean"] / eo["resid_mean"] - 1) < 1e-8 and abs(eg["rz"] / eo["rz"] - 1) < 1e-8
    (mg, ag), (mo, ao) = g.state(), o.state()
    assert np.linalg.norm(mg - mo) <= 1e-10 * np.linalg.norm(mo)
    assert np.linalg.norm(ag - ao) <= 1e-10 * np.linalg.norm(ao)
    assert [r[0] for r in g.reports()] == [r[0] for r in o.reports()]
