"""Edge cases of the relaxation path against the reference itself (oracle/_ref):
zero and non-finite right-hand sides (sparse.hpp:305-309, 323-324), a single sweep
(max_iter = 1), the smallest meshes (one hex cell / one cube of 6 tets: rows padded
inside a 32-row SELL slice, ragged degrees), every sweep kernel variant."""
import numpy as np
import pytest

from paper_2404_01407_b200.mesh import structured_sector

pytestmark = pytest.mark.gpu

PATHS = [("rb-exact", True, 0), ("rb-split", True, 1), ("level", False, 0)]


def _set_path(la, rb, mode):
    la.set_red_black(rb)
    la.set_rb_sweep(mode)


@pytest.fixture(autouse=True)
def _restore():
    yield
    from paper_2404_01407_b200 import la
    _set_path(la, True, la.RB_EXACT)


def _sys(m, b, seed, cplx):
    rng = np.random.default_rng(seed)
    pat = m.pattern(b)
    A = rng.standard_normal((len(pat["col_idx"]), b, b)) * 0.1
    A[pat["diag_idx"]] += np.eye(b) * 4
    shift = rng.uniform(0.5, 2, m.n) if cplx else None
    Aref = A.astype(np.complex128) if cplx else A
    if cplx:
        Aref[pat["diag_idx"]] += 1j * np.eye(b) * shift[:, None, None]
    return pat, A.reshape(-1), shift, Aref.reshape(-1), rng


MESHES = {"hex1": dict(cells=(1, 1, 1)), "hex3x2x1": dict(cells=(3, 2, 1)),
          "tet1": dict(cells=(1, 1, 1), tets=True), "tet2x2x1": dict(cells=(2, 2, 1), tets=True, jitter=0.05)}


@pytest.mark.parametrize("mesh", list(MESHES))
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("path", PATHS, ids=[p[0] for p in PATHS])
def test_smallest_meshes_and_single_sweep(ref, mesh, cplx, path):
    from paper_2404_01407_b200 import la
    kw = dict(MESHES[mesh])
    m = structured_sector(*kw.pop("cells"), seed=3, **kw)
    b = 5
    pat, A, shift, Aref, rng = _sys(m, b, 11 + cplx, cplx)
    P = la.Pattern.from_dict(pat)
    _set_path(la, path[1], path[2])
    rhs = rng.standard_normal(m.n * b) + (1j * rng.standard_normal(m.n * b) if cplx else 0)
    for tol, it in ((0.5, 1), (1e-12, 1), (1e-12, 3)):
        xr, rr = ref.smoothed_solve(pat, Aref, rhs, tol, it)
        xd, rd = la.smoothed_solve(P, A, rhs, tol, it, shift) if cplx else la.smoothed_solve(P, A, rhs, tol, it)
        assert rd[0] == rr[0] and rd[3] == rr[3], (rd, rr)
        assert np.array_equal(xd, xr)
        assert abs(rd[1] / rr[1] - 1) < 1e-14 and abs(rd[2] / rr[2] - 1) < 1e-12


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("path", PATHS, ids=[p[0] for p in PATHS])
def test_zero_rhs_converges_without_sweeping(ref, cplx, path):
    """||b|| = 0: zero iterations, converged, x = 0 (sparse.hpp:305-309)."""
    from paper_2404_01407_b200 import la
    m = structured_sector(6, 4, 3, seed=2)
    pat, A, shift, Aref, _ = _sys(m, 5, 5, cplx)
    P = la.Pattern.from_dict(pat)
    _set_path(la, path[1], path[2])
    rhs = np.zeros(m.n * 5, np.complex128 if cplx else np.float64)
    xr, rr = ref.smoothed_solve(pat, Aref, rhs, 1e-2, 5)
    xd, rd = la.smoothed_solve(P, A, rhs, 1e-2, 5, shift) if cplx else la.smoothed_solve(P, A, rhs, 1e-2, 5)
    assert rr == (0, 0.0, 0.0, True) and rd == rr
    assert not np.any(xd) and not np.any(xr)


@pytest.mark.parametrize("bad", [np.nan, np.inf])
@pytest.mark.parametrize("path", PATHS, ids=[p[0] for p in PATHS])
def test_non_finite_rhs_raises_divergence(ref, bad, path):
    """A non-finite iterate throws DivergenceError at the first sweep (sparse.hpp:323-324),
    on the device as in the reference."""
    from paper_2404_01407_b200 import la
    from paper_2404_01407_b200._lib import FnlhError
    m = structured_sector(6, 4, 3, seed=2)
    pat, A, shift, Aref, rng = _sys(m, 5, 6, True)
    P = la.Pattern.from_dict(pat)
    _set_path(la, path[1], path[2])
    rhs = rng.standard_normal(m.n * 5) + 0j
    rhs[17] = bad
    with pytest.raises(Exception, match="DivergenceError"):
        ref.smoothed_solve(pat, Aref, rhs, 1e-2, 5)
    with pytest.raises(FnlhError) as ei:
        la.smoothed_solve(P, A, rhs, 1e-2, 5, shift)
    assert ei.value.kind == "DivergenceError"
