"""CPU: the synthetic BASELINE inputs (mesh generators, orderings, seeded cases)."""
import numpy as np
import pytest

from paper_2404_01407_b200.cases import SPECS, make_case
from paper_2404_01407_b200.mesh import structured_sector


def test_c1_counts_match_survey_table():
    """C1 periodic 32x16x8 -> N 4,752, E 13,584, nnzb 31,920."""
    m = structured_sector(32, 16, 8, geometry="channel", periodic_j=True)
    pat = m.pattern()
    assert m.n == 4752
    assert (m.fbc < 0).sum() == 13584
    assert len(pat["col_idx"]) == 31920


@pytest.mark.parametrize("tets", [False, True])
def test_median_dual_closure(tets):
    """Interior dual cells are closed: the closure vector vanishes away from walls; the
    total closure equals -(inlet + outlet) areas = 0 in x and the wall force elsewhere."""
    m = structured_sector(8, 6, 5, tets=tets, jitter=0.05 if tets else 0.0, seed=3)
    c = m.closure.reshape(-1, 3)
    X = m.coords
    r = np.sqrt(X[:, 1] ** 2 + X[:, 2] ** 2)
    th = np.arctan2(X[:, 2], X[:, 1])
    interior = ((r > 0.5 + 1e-9) & (r < 1.0 - 1e-9) & (th > 1e-9) & (th < np.deg2rad(10) - 1e-9)
                & (m.bflag == 0))
    assert interior.sum() > 0
    scale = np.abs(m.fn).max()
    assert np.abs(c[interior]).max() < 1e-12 * scale * 10
    assert np.all(m.vol > 0) and np.all(m.farea > 0)


@pytest.mark.parametrize("tets,ncol", [(False, 2), (True, 8)])
def test_colour_major_ordering(tets, ncol):
    m = structured_sector(6, 5, 4, tets=tets, jitter=0.05 if tets else 0.0, seed=2)
    assert np.all(np.diff(m.colour) >= 0)
    assert len(np.unique(m.colour)) == ncol
    inter = m.fbc < 0
    assert not np.any(m.colour[m.fa[inter]] == m.colour[m.fb[inter]])


@pytest.mark.parametrize("order", ["rcm", "morton", "lex", "lexk"])
def test_orders_inside_a_colour_keep_the_ilu_pattern(order):
    """The numbering inside each colour is free on a 2-colour ordering: every order is
    colour-major, a permutation of the same nodes, with the same geometry per node."""
    m = structured_sector(9, 7, 5, seed=2, order=order)
    ref = structured_sector(9, 7, 5, seed=2, order="rcm")
    assert (np.diff(m.colour) >= 0).all() and (m.colour == ref.colour).all()
    key = lambda q: sorted(map(tuple, np.round(q.coords, 12)))  # noqa: E731
    assert key(m) == key(ref)
    ia = np.lexsort(np.round(m.coords, 12).T)
    ib = np.lexsort(np.round(ref.coords, 12).T)
    assert np.array_equal(m.vol[ia], ref.vol[ib])
    pat = m.pattern()
    assert len(pat["col_idx"]) == len(ref.pattern()["col_idx"])


def test_node_face_csr_ascending():
    m = structured_sector(5, 4, 3, seed=5)
    for i in range(m.n):
        f = m.nf_idx[m.nf_ptr[i]:m.nf_ptr[i + 1]]
        assert np.all(np.diff(f) > 0)


def test_cases_are_seeded_and_deterministic():
    a = make_case("c1", scale=0.5)
    b = make_case("c1", scale=0.5)
    assert np.array_equal(a.mean0, b.mean0) and np.array_equal(a.forcing, b.forcing)
    assert np.array_equal(a.mesh.fn, b.mesh.fn)
    assert set(SPECS) == {"c1", "c2", "c3", "c4", "c5"}


def test_c5_has_sa_scalar_and_eddy_viscosity():
    c = make_case("c5", scale=0.06)
    assert c.mesh.b == 6
    assert c.mesh.mu.min() >= 1e-6 and c.mesh.mu.max() <= 1e-3


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_agglomeration_hierarchy(name):
    """2x2x2 agglomeration (mesh.coarsen, the 3D counterpart of multigrid.cpp:9-127):
    volumes, closures and boundary areas are conserved level to level, every coarse node
    has at most 8 children, and the coarse forcing is the children's area-weighted mean."""
    from paper_2404_01407_b200.mesh import hierarchy
    c = make_case(name, scale=0.08)
    h = hierarchy(c.mesh, 3, c.forcing)
    for lv in range(2):
        mf, par, ff = h[lv]
        mc, _, fc = h[lv + 1]
        assert par.min() == 0 and par.max() == mc.n - 1
        assert np.bincount(par).max() <= 8
        vs = np.zeros(mc.n)
        np.add.at(vs, par, mf.vol)
        assert np.array_equal(vs, mc.vol)
        cl = np.zeros((mc.n, 3))
        np.add.at(cl, par, mf.closure.reshape(-1, 3))
        scale = np.abs(mf.fn).max()
        assert np.abs(cl - mc.closure.reshape(-1, 3)).max() < 1e-12 * scale
        for kind in (0, 1):
            af = mf.farea[mf.fbc == kind].sum()
            ac = mc.farea[mc.fbc == kind].sum()
            assert ac <= af * (1 + 1e-12)  # summed normals: equal on planar patches
        assert fc.shape == (len(c.forcing), 3 * mc.n_boundary)
        # a uniform forcing stays uniform
        assert np.abs(np.abs(fc[:, 3 * np.flatnonzero(mc.fbc[mc.fbc >= 0] == 0) + 1]) - 1e-3 / 1.4).max() < 1e-15
    assert h[2][1] is None


def test_hierarchy_needs_structure():
    from paper_2404_01407_b200.mesh import hierarchy
    c = make_case("c1", scale=0.25)
    c.mesh.ijk = None
    with pytest.raises(ValueError):
        hierarchy(c.mesh, 2)
    assert len(hierarchy(c.mesh, 1)) == 1
