"""Pin the C restatement (oracle/fnlh_oracle.c) against the reference itself
(oracle/_ref/libfnlh_ref.so, the unmodified /root/reference sources).

Generic layers must be bitwise; the 3D discretization on the reference nozzle's line
mesh must be bitwise at first order (FD Jacobian, face_flux1) and within 1e-13 at
second order (the edge-based JST Laplacian re-associates the 1D 4th difference)."""
import numpy as np
import pytest

from helpers import (NOZZLE_CASE, embed, extract, extract_blocks, forcing_triplets, line_mesh_from_ref, rel)
from paper_2404_01407_b200._lib import pow_mode
from paper_2404_01407_b200.mesh import structured_sector


def _random_system(m, b, rng, cplx):
    pat = m.pattern(b)
    nnzb = len(pat["col_idx"])
    A = rng.standard_normal((nnzb, b, b)) * 0.1
    A[pat["diag_idx"]] += np.eye(b) * 4
    if cplx:
        A = A + 0j
        A[pat["diag_idx"]] += 1j * np.eye(b) * rng.uniform(0.5, 2, m.n)[:, None, None]
    return pat, A.reshape(-1)


@pytest.mark.parametrize("b", [1, 3, 5, 6])
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("tets", [False, True])
def test_ilu_and_richardson_bitwise(ref, orc, b, cplx, tets):
    rng = np.random.default_rng(b + 10 * cplx + 100 * tets)
    m = structured_sector(6, 5, 4, tets=tets, jitter=0.05 if tets else 0.0, seed=3)
    pat, A = _random_system(m, b, rng, cplx)
    fr, fo = ref.ilu_factorize(pat, A), orc.ilu_factorize(pat, A)
    for k in fr:
        assert np.array_equal(fr[k], fo[k]), k
    rhs = rng.standard_normal(m.n * b) + (1j * rng.standard_normal(m.n * b) if cplx else 0)
    xr, rr = ref.smoothed_solve(pat, A, rhs, 1e-8, 10)
    xo, ro = orc.smoothed_solve(pat, A, rhs, 1e-8, 10)
    assert np.array_equal(xr, xo) and rr == ro


def test_partition_dropping_bitwise(ref, orc):
    rng = np.random.default_rng(7)
    m = structured_sector(6, 5, 4, seed=1)
    pat, A = _random_system(m, 5, rng, True)
    pat["partition"] = (np.arange(m.n) * 4 // m.n).astype(np.int32)
    fr, fo = ref.ilu_factorize(pat, A), orc.ilu_factorize(pat, A)
    for k in fr:
        assert np.array_equal(fr[k], fo[k]), k


def test_build_lhs_mean_bitwise(ref, orc):
    rng = np.random.default_rng(2)
    m = structured_sector(4, 4, 3, seed=2)
    pat = m.pattern()
    J = rng.standard_normal(len(pat["col_idx"]) * 25)
    for implicit in (0, 1):
        for stage in (1, 3, 5):
            assert np.array_equal(ref.build_lhs_mean(pat, J, implicit, 50.0, 0.6, stage),
                                  orc.build_lhs_mean(pat, J, implicit, 50.0, 0.6, stage))


def test_smith_division_is_libgcc(ref):
    """The device complex division (Smith's method, normal range) reproduces the
    reference's std::complex<double> division (libgcc __divdc3) bit for bit."""
    rng = np.random.default_rng(0)
    a = rng.standard_normal(20000) + 1j * rng.standard_normal(20000)
    b = (rng.standard_normal(20000) + 1j * rng.standard_normal(20000)) * 10.0 ** rng.uniform(-3, 3, 20000)
    q = ref.cdiv(a, b)
    ar, ai, br, bi = a.real, a.imag, b.real, b.imag
    m = np.abs(br) < np.abs(bi)
    ratio = np.where(m, br / bi, bi / br)
    den = np.where(m, br * ratio + bi, bi * ratio + br)
    xr = np.where(m, (ar * ratio + ai) / den, (ai * ratio + ar) / den)
    xi = np.where(m, (ai * ratio - ar) / den, (ai - ar * ratio) / den)
    assert np.array_equal(xr + 1j * xi, q)


@pytest.fixture(scope="module")
def nozzle(ref):
    noz = ref.nozzle(NOZZLE_CASE.format(nx=64, nh=2))
    rng = np.random.default_rng(0)
    W3 = noz.initial_mean().reshape(-1, 3)
    W3 = (W3 * (1 + 0.01 * rng.uniform(-1, 1, W3.shape))).reshape(-1)
    what3 = (rng.standard_normal(noz.n * 3) + 1j * rng.standard_normal(noz.n * 3)) * 1e-3 * np.tile(
        np.abs(W3.reshape(-1, 3)).mean(0), noz.n)
    return noz, line_mesh_from_ref(noz), W3, what3


def test_nozzle_first_order_bitwise(nozzle, orc):
    noz, m, W3, _ = nozzle
    W5 = embed(W3, noz.n)
    ri, _ = noz.residual(W3, 1)
    oi, _ = orc.residual(m, W5, 1)
    assert np.array_equal(extract(oi, noz.n), ri)
    J5, _ = orc.fd_jacobian(m, noz.pattern(5), W5)
    assert np.array_equal(extract_blocks(J5, noz.nnzb), noz.jacobian(W3))
    _, P5 = orc.fd_jacobian(m, noz.pattern(5), W5, want_J=False, want_P=True)
    assert np.array_equal(extract_blocks(P5, noz.n), noz.diag_blocks(W3))


def test_nozzle_second_order_and_perturbation(nozzle, orc):
    noz, m, W3, what3 = nozzle
    W5 = embed(W3, noz.n)
    ri, _ = noz.residual(W3, 2)
    oi, _ = orc.residual(m, W5, 2)
    assert np.array_equal(extract(oi, noz.n), ri)  # the 1D stencil on line meshes (disc_euler.cpp:113-157)
    f3 = np.array([1.0, -2.0, 30.0])
    Wp = W3 * 1.0001
    ri, _ = noz.residual(Wp, 2, mode=1, wref=W3, forcing=f3)
    oi, _ = orc.residual(m, embed(Wp, noz.n), 2, mode=1, wref=embed(W3, noz.n), forcing=forcing_triplets(f3))
    assert np.array_equal(extract(oi, noz.n), ri)


def test_nozzle_linearized_residual_and_df(nozzle, orc):
    noz, m, W3, what3 = nozzle
    W5 = embed(W3, noz.n)
    f3 = noz.forcing[0]
    ri, _ = noz.linearized_residual(W3, what3, noz.omega[0], f3)
    oi, _ = orc.linearized_residual(m, W5, embed(what3, noz.n, np.complex128), noz.omega[0], forcing_triplets(f3))
    assert np.array_equal(extract(oi, noz.n), ri)
    amps3 = np.stack([what3, 0.5 * what3])
    df3 = noz.deterministic_flux(W3, noz.omega, amps3)
    df5 = orc.deterministic_flux(m, W5, noz.omega, np.stack([embed(a, noz.n, np.complex128) for a in amps3]))
    assert np.array_equal(extract(df5, noz.n), df3)


def test_nozzle_solver_history(ref, orc):
    """Full FnlhSolver (driver.cpp:157-333) vs the restated outer iteration, 20 steps: with
    the reference's own 1D JST stencil on the line mesh and glibc's pow the restatement is
    the reference bit for bit (states equal; the RMS differ only by the sqrt(5/3) rescaling
    of the b = 5 embedding)."""
    case = NOZZLE_CASE.format(nx=64, nh=2)
    rs = ref.solver(case)
    noz = rs.noz
    m = line_mesh_from_ref(noz)
    forc = np.stack([forcing_triplets(f) for f in noz.forcing])
    osv = orc.solver(m, noz.pattern(5), dict(implicit=1), noz.omega, forc, embed(noz.initial_mean(), noz.n))
    s = np.sqrt(5 / 3)  # RMS over n*b dofs: b = 5 here, 3 in the reference
    for it in range(20):
        er, eo = rs.outer_iteration(), osv.outer_iteration()
        assert abs(eo["resid_mean"] * s / er["resid_mean"] - 1) < 1e-14, (it, eo, er)
        assert abs(eo["rz"] * s / er["rz"] - 1) < 1e-14, (it, eo, er)
    mr, ar = rs.state()
    mo, ao = osv.state()
    assert np.array_equal(extract(mo, noz.n), mr)
    assert np.array_equal(np.stack([extract(a, noz.n) for a in ao]), ar)


def test_oracle_harmonic_workers_bitwise():
    """The checker's harmonic worker threads (the reference's workers, driver.cpp:246-265,
    used by the CPU baseline) give bitwise the sequential result."""
    from oracle.oracle import Oracle
    from paper_2404_01407_b200.cases import make_case
    c = make_case("c2", scale=0.05, nh=3)
    out = []
    for w in (1, 3):
        s = Oracle(pow_mode=pow_mode(), workers=w).solver(c.mesh, c.mesh.pattern(), c.scheme, c.omegas, c.forcing, c.mean0)
        hist = [s.outer_iteration() for _ in range(2)]
        out.append(([(e["resid_mean"], e["rz"]) for e in hist], s.state(), s.reports()))
    (h1, (m1, a1), r1), (h3, (m3, a3), r3) = out
    assert h1 == h3 and r1 == r3
    assert np.array_equal(m1, m3) and np.array_equal(a1, a3)


@pytest.mark.parametrize("levels", [1, 2, 3])
def test_nozzle_explicit_multigrid_history(ref, orc, levels):
    """The explicit scheme with the FAS V-cycle (multigrid.cpp:142-232, driver.cpp:223-241,
    297-311): the reference's FnlhSolver with mg_levels vs the restated hierarchy built by
    mesh.hierarchy on the embedded line mesh (pairwise agglomeration: the reference's
    coarse meshes, forcing and parent maps)."""
    from paper_2404_01407_b200.mesh import hierarchy
    case = NOZZLE_CASE.format(nx=64, nh=2)
    rs = ref.solver(case, implicit=0, mg_levels=levels, sigma=1.0)  # CFL 2 diverges on this nozzle
    noz = rs.noz
    m = line_mesh_from_ref(noz)
    m.ijk = np.stack([np.arange(noz.n), np.zeros(noz.n, np.int64), np.zeros(noz.n, np.int64)], axis=1)
    forc = np.stack([forcing_triplets(f) for f in noz.forcing])
    hier = hierarchy(m, levels, forc)
    osv = orc.solver(m, noz.pattern(5), dict(implicit=0, sigma_cfl=1.0), noz.omega, forc,
                     embed(noz.initial_mean(), noz.n))
    for lv in range(1, levels):
        mc, _, fc = hier[lv]
        osv.add_level(mc, hier[lv - 1][1], fc)
        assert mc.n == noz.n >> lv
    s = np.sqrt(5 / 3)
    for it in range(10):
        er, eo = rs.outer_iteration(), osv.outer_iteration()
        assert abs(eo["resid_mean"] * s / er["resid_mean"] - 1) < 1e-14, (it, eo, er)
        assert abs(eo["rz"] * s / er["rz"] - 1) < 1e-14, (it, eo, er)
    mr, ar = rs.state()
    mo, ao = osv.state()
    assert np.array_equal(extract(mo, noz.n), mr)
    assert np.array_equal(np.stack([extract(a, noz.n) for a in ao]), ar)
