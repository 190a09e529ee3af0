"""Mesh preprocessing.  CPU: the host restatement of the pattern and
adjacency builders against the reference's own make_pattern (sparse.cpp:91-117) and
Mesh::build_adjacency (mesh.cpp:44-59).  GPU: the device builders (csrc/meshgen.cu)
bitwise against the host restatement (mesh.py)."""
import numpy as np
import pytest

from paper_2404_01407_b200.mesh import structured_sector

GEOMS = [dict(tets=False), dict(tets=True, jitter=0.05), dict(tets=False, periodic_j=True, geometry="channel"),
         dict(tets=True, periodic_j=True, geometry="channel")]
FIELDS = ("fa", "fb", "fbc", "ford", "fn", "farea", "fnh", "fvis", "vol", "closure", "mu", "nf_ptr", "nf_idx",
          "bflag", "colour", "coords", "ijk")


@pytest.mark.parametrize("kw", GEOMS)
def test_host_pattern_and_adjacency_match_reference(ref, kw):
    m = structured_sector(7, 6, 5, seed=4, device=False, **kw)
    inner = m.fbc < 0
    pr = ref.make_pattern(5, m.n, m.fa[inner], m.fb[inner])
    ph = m.pattern(device=False)
    for k in ("row_ptr", "col_idx", "diag_idx"):
        assert np.array_equal(pr[k], ph[k]), k
    fb = np.where(inner, m.fb, -1)
    nf_ptr, nf_idx = ref.build_adjacency(m.n, m.fa, fb)
    assert np.array_equal(nf_ptr, m.nf_ptr) and np.array_equal(nf_idx, m.nf_idx)


def test_pattern_edge_cases(ref):
    """duplicate edges, self loops and isolated rows (make_pattern sorts and uniques)."""
    ea = np.array([0, 3, 3, 2, 4], np.int32)
    eb = np.array([3, 0, 3, 4, 2], np.int32)
    pr = ref.make_pattern(2, 6, ea, eb)
    assert list(pr["row_ptr"]) == [0, 2, 3, 5, 7, 9, 10]
    assert list(pr["col_idx"]) == [0, 3, 1, 2, 4, 0, 3, 2, 4, 5]


@pytest.mark.gpu
@pytest.mark.parametrize("kw", GEOMS)
def test_device_sector_bitwise(kw):
    a = structured_sector(9, 8, 6, seed=7, device=False, **kw)
    b = structured_sector(9, 8, 6, seed=7, device=True, **kw)
    for f in FIELDS:
        va, vb = getattr(a, f), getattr(b, f)
        assert (va is None and vb is None) or np.array_equal(va, vb), f
    pa, pb = a.pattern(device=False), b.pattern(device=True)
    for k in ("row_ptr", "col_idx", "diag_idx", "partition"):
        assert np.array_equal(pa[k], pb[k]), k


@pytest.mark.gpu
def test_device_pattern_edge_cases(ref):
    from paper_2404_01407_b200.mesh import make_pattern_device
    from paper_2404_01407_b200._lib import FnlhError
    ea = np.array([0, 3, 3, 2, 4], np.int32)
    eb = np.array([3, 0, 3, 4, 2], np.int32)
    pr = ref.make_pattern(2, 6, ea, eb)
    pd = make_pattern_device(6, ea, eb, 2)
    for k in ("row_ptr", "col_idx", "diag_idx"):
        assert np.array_equal(pr[k], pd[k]), k
    pd0 = make_pattern_device(3, np.zeros(0, np.int32), np.zeros(0, np.int32), 1)
    assert list(pd0["row_ptr"]) == [0, 1, 2, 3] and list(pd0["col_idx"]) == [0, 1, 2]
    with pytest.raises(FnlhError, match="out of range"):
        make_pattern_device(3, np.array([0], np.int32), np.array([5], np.int32), 1)


@pytest.mark.gpu
def test_device_sector_c4_size():
    """The C4 mesh (4.3 M nodes) through the device path; spot-checks of the invariants."""
    import time
    t = time.time()
    m = structured_sector(256, 128, 128, seed=404, device=True)
    dt = time.time() - t
    assert m.n == 257 * 129 * 129
    assert (m.vol > 0).all() and (m.farea > 0).all()
    print(f"C4 sector mesh on the device: {dt:.1f} s")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["hex", "tet", "periodic", "components"])
def test_device_rcm_equals_scipy(kind):
    """fnlh_rcm (level-synchronous Cuthill-McKee on the device) reproduces
    scipy.sparse.csgraph.reverse_cuthill_mckee exactly: hex / jittered-tet / periodic sector
    graphs in a seeded random numbering, and a graph of several components (starts by
    ascending degree, stable)."""
    from paper_2404_01407_b200.mesh import rcm_order, structured_sector
    rng = np.random.default_rng(17)
    if kind == "components":
        n = 300
        ea = rng.integers(0, n, 500)
        eb = rng.integers(0, n, 500)
        keep = (ea != eb) & ((ea < 100) == (eb < 100)) & ((ea < 200) == (eb < 200))
        ea, eb = ea[keep], eb[keep]
    else:
        kw = dict(tets=True, jitter=0.05) if kind == "tet" else dict(periodic_j=True) if kind == "periodic" else {}
        m = structured_sector(12, 8, 6, seed=2, **kw)
        inter = m.fbc < 0
        p = rng.permutation(m.n)
        n, ea, eb = m.n, p[m.fa[inter]], p[m.fb[inter]]
    assert np.array_equal(rcm_order(n, ea, eb, device=True), rcm_order(n, ea, eb, device=False))


@pytest.mark.gpu
def test_device_rcm_c4_size():
    """The full C4 graph (4.28 M nodes, 12.7 M edges): equal to scipy."""
    import time
    from paper_2404_01407_b200.mesh import rcm_order, _sector_dual_device, structured_sector  # noqa: F401
    ci, cj, ck = 256, 128, 128
    ni, nj, nk = ci + 1, cj + 1, ck + 1
    idx = np.arange(ni * nj * nk).reshape(ni, nj, nk)
    ea = np.concatenate([idx[:-1].ravel(), idx[:, :-1].ravel(), idx[:, :, :-1].ravel()])
    eb = np.concatenate([idx[1:].ravel(), idx[:, 1:].ravel(), idx[:, :, 1:].ravel()])
    p = np.random.default_rng(3).permutation(idx.size)
    t0 = time.time()
    d = rcm_order(idx.size, p[ea], p[eb], device=True)
    t1 = time.time()
    h = rcm_order(idx.size, p[ea], p[eb], device=False)
    t2 = time.time()
    print(f"rcm at C4 size: device {t1 - t0:.2f} s, scipy {t2 - t1:.2f} s")
    assert np.array_equal(d, h)
