"""Shared test helpers: the reference nozzle embedded as a 3D line mesh (b = 5).

The reference's quasi-1D nozzle (disc_euler.cpp) is the special case of the 3D
edge-based discretization with face normals (A, 0, 0): these helpers build that line
mesh from the reference's own mesh arrays and map states between b = 3
(rho, u, p) and b = 5 (rho, u, v=0, w=0, p)."""
import numpy as np

from paper_2404_01407_b200.mesh import from_faces

IDX3 = np.array([0, 1, 4])


def nozzle_from_golden(path):
    """RefNozzle-like view of tests/golden/nozzle_nx64_h2.npz (no reference needed)."""
    import types
    g = np.load(path, allow_pickle=False)
    gas = g["gas"]
    ns = types.SimpleNamespace(**{k: g[k] for k in g.files})
    ns.n = int(g["n"])
    ns.nf = len(g["fa"])
    ns.nnzb = len(g["col_idx"])
    ns.gamma, ns.gas_constant, ns.p0, ns.T0, ns.p_out, ns.forcing_scale = [float(v) for v in gas]

    def pattern(b=3):
        diag = np.array([ns.row_ptr[i] + np.searchsorted(ns.col_idx[ns.row_ptr[i]:ns.row_ptr[i + 1]], i)
                         for i in range(ns.n)], np.int32)
        return dict(b=b, row_ptr=ns.row_ptr, col_idx=ns.col_idx, diag_idx=diag, partition=np.zeros(ns.n, np.int32))
    ns.pattern = pattern
    return ns


def line_mesh_from_ref(noz):
    nf = noz.nf
    fn = np.zeros((nf, 3))
    sign = np.where(noz.fbc == 0, -1.0, 1.0)      # west boundary faces point to -x
    fn[:, 0] = sign * noz.area
    fbc = np.where(noz.fbc < 0, -1, noz.fbc).astype(np.int32)
    ford = np.zeros(nf, np.int32)
    bidx = np.flatnonzero(fbc >= 0)
    ford[bidx] = np.arange(len(bidx))
    m = from_faces(noz.n, noz.fa, noz.fb, fbc, ford, fn, noz.vol, b=5, gamma=noz.gamma,
                   gas_constant=noz.gas_constant, p0=noz.p0, T0=noz.T0, p_out=noz.p_out,
                   forcing_scale=noz.forcing_scale)
    assert np.array_equal(m.nf_ptr, noz.nf_ptr) and np.array_equal(m.nf_idx, noz.nf_idx)
    return m


def embed(v3, n, dtype=np.float64):
    v = np.zeros((n, 5), dtype)
    v[:, IDX3] = np.asarray(v3).reshape(n, 3)
    return v.reshape(-1)


def extract(v5, n):
    return np.asarray(v5).reshape(n, 5)[:, IDX3].reshape(-1)


def forcing_triplets(f3, nbfaces=2):
    return np.tile(np.asarray(f3), nbfaces)


def extract_blocks(J5, nblocks):
    J = np.asarray(J5).reshape(nblocks, 5, 5)
    return J[:, IDX3][:, :, IDX3].reshape(-1)


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


NOZZLE_CASE = "kind = nozzle-euler\nnx = {nx}\nharmonics = {nh}\nbase_omega = 500\n"


def assert_reports_match(ra, rb, tol=1e-14):
    """Linear-solve reports of two runs whose harmonics ran in different lane batches: the
    iteration counts and convergence flags equal, the norms to `tol` (the 2-colour sweep sums
    its CTA partials over row blocks whose size depends on the lane count, rb.cuh)."""
    assert len(ra) == len(rb)
    assert [(r[0], r[3]) for r in ra] == [(r[0], r[3]) for r in rb]
    for a, b in zip(ra, rb):
        assert abs(a[1] - b[1]) <= tol * abs(a[1]) and abs(a[2] - b[2]) <= tol * abs(a[2]), (a, b)
