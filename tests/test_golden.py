"""CPU: the restatement against golden vectors produced by the reference itself
(tests/golden/make_golden.py ran oracle/_ref/libfnlh_ref.so).  Runs without
/root/reference, so it also pins the oracle on the GPU box."""
import os

import numpy as np
import pytest

from helpers import embed, extract, extract_blocks, forcing_triplets, line_mesh_from_ref, nozzle_from_golden, rel

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def noz():
    return nozzle_from_golden(os.path.join(GOLD, "nozzle_nx64_h2.npz"))


@pytest.fixture(scope="module")
def la_gold():
    return np.load(os.path.join(GOLD, "la_hex4x3x3.npz"))


def test_nozzle_first_order_and_jacobian_bitwise(orc, noz):
    m = line_mesh_from_ref(noz)
    W5 = embed(noz.W3, noz.n)
    oi, _ = orc.residual(m, W5, 1)
    assert np.array_equal(extract(oi, noz.n), noz.res1)
    J5, _ = orc.fd_jacobian(m, noz.pattern(5), W5)
    assert np.array_equal(extract_blocks(J5, noz.nnzb), noz.J)


def test_nozzle_second_order_linres_df(orc, noz):
    m = line_mesh_from_ref(noz)
    W5 = embed(noz.W3, noz.n)
    oi, _ = orc.residual(m, W5, 2)
    assert np.array_equal(extract(oi, noz.n), noz.res2)
    li, _ = orc.linearized_residual(m, W5, embed(noz.what3, noz.n, np.complex128), noz.omega[0],
                                    forcing_triplets(noz.forcing[0]))
    assert np.array_equal(extract(li, noz.n), noz.linres)
    amps = np.stack([embed(noz.what3, noz.n, np.complex128), embed(0.5 * noz.what3, noz.n, np.complex128)])
    df = orc.deterministic_flux(m, W5, noz.omega, amps)
    assert np.array_equal(extract(df, noz.n), noz.df)


def test_nozzle_history(orc, noz):
    """FnlhSolver history (driver.cpp:157-333): 20 outer iterations of the reference."""
    m = line_mesh_from_ref(noz)
    forc = np.stack([forcing_triplets(f) for f in noz.forcing])
    s = orc.solver(m, noz.pattern(5), dict(implicit=1), noz.omega, forc, embed(noz.mean0, noz.n))
    k = np.sqrt(5 / 3)
    for it in range(20):
        e = s.outer_iteration()
        assert abs(e["resid_mean"] * k / noz.hist[it, 1] - 1) < 1e-14
        assert abs(e["rz"] * k / noz.hist[it, 2] - 1) < 1e-14
    mean, amps = s.state()
    assert np.array_equal(extract(mean, noz.n), noz.mean20)
    assert np.array_equal(np.stack([extract(a, noz.n) for a in amps]), noz.amps20)


def test_nozzle_run_policy(noz):
    """Linear-solve policy (SPEC.md acceptance 8): every solve reaches 1e-2 or stops at 10."""
    reps = noz.run_reports
    assert len(reps) > 0
    assert np.all((reps[:, 2] <= 1e-2 * reps[:, 1]) | (reps[:, 0] == 10))


@pytest.mark.parametrize("key", ["b5_z", "b5_d", "b3_z"])
def test_la_bitwise(orc, la_gold, key):
    g = la_gold
    b = int(key[1])
    cplx = key.endswith("z")
    from paper_2404_01407_b200.mesh import structured_sector
    m = structured_sector(4, 3, 3, seed=11)
    pat = m.pattern(b)
    assert np.array_equal(pat["row_ptr"], g["row_ptr"]) and np.array_equal(pat["col_idx"], g["col_idx"])
    A = g[f"{key}_A"]
    if cplx:
        Az = A.reshape(-1, b, b).astype(np.complex128)
        Az[pat["diag_idx"]] += 1j * np.eye(b) * g[f"{key}_shift"][:, None, None]
        A = Az.reshape(-1)
    f = orc.ilu_factorize(pat, A)
    for k in ("vals", "diag_lu", "diag_piv", "diag_inv"):
        assert np.array_equal(f[k], g[f"{key}_{k}"]), k
    x, rep = orc.smoothed_solve(pat, A, g[f"{key}_rhs"], 1e-6, 6)
    assert np.array_equal(x, g[f"{key}_x"])
    assert rep[0] == int(g[f"{key}_rep"][0])
