"""Node-centred median-dual meshes for the 3D edge-based FNLH discretization.

The reference meshes are 1D/2D with axis-aligned faces carrying a scalar area
(``mesh.hpp:24-62``).  The BASELINE configurations are 3D hex / Kuhn-tet sectors,
so a face here carries an area-weighted normal ``fn`` (a -> b for interior edges,
outward on inlet/outlet faces).  Slip walls are not faces: their pressure force is
the node closure source ``-p * closure_i`` (``closure_i`` = sum of the node's
incident outward normals), which is exactly the reference nozzle's area source
``-p (A_R - A_L)`` (``disc_euler.cpp:95-100``) on a line mesh.

Node ordering (the ILU(0) order): seeded random permutation -> reverse
Cuthill-McKee -> stable colour-major sort, so ILU(0) rows of one colour are
independent and the device factorizes / substitutes colour by colour while staying
the reference's natural-order algorithm (``sparse.cpp:187-291``) on this ordering.
"""
from __future__ import annotations

import dataclasses
import itertools

import numpy as np


@dataclasses.dataclass
class Mesh3D:
    n: int
    nf: int
    b: int
    fa: np.ndarray        # int32 [nf]
    fb: np.ndarray        # int32 [nf], -1 on boundary faces
    fbc: np.ndarray       # int32 [nf], -1 interior, 0 inlet (west), 1 outlet (east)
    ford: np.ndarray      # int32 [nf], global boundary ordinal (forcing slot), 0 interior
    fn: np.ndarray        # float64 [nf*3]
    farea: np.ndarray     # float64 [nf]
    fnh: np.ndarray       # float64 [nf*3]
    fvis: np.ndarray      # float64 [nf]
    vol: np.ndarray       # float64 [n]
    closure: np.ndarray   # float64 [n*3]
    mu: np.ndarray        # float64 [n]
    nf_ptr: np.ndarray    # int32 [n+1]
    nf_idx: np.ndarray    # int32
    bflag: np.ndarray     # int32 [n]
    gamma: float = 1.4
    gas_constant: float = 287.05
    p0: float = 101325.0
    T0: float = 300.0
    p_out: float = 98000.0
    nt_in: float = 0.0
    forcing_scale: float = 98000.0
    colour: np.ndarray | None = None       # int32 [n], nondecreasing in colour-major orders
    partition: np.ndarray | None = None    # int32 [n]
    coords: np.ndarray | None = None       # float64 [n,3]
    n_boundary: int = 0
    ijk: np.ndarray | None = None          # int64 [n,3] structured indices (coarsening), if any

    # --- sparsity pattern of the block LHS (sparse.cpp:61-117): adjacency + diagonal
    def pattern(self, b: int | None = None, device: bool | None = None):
        n = self.n
        interior = self.fbc < 0
        if device is None:
            device = _device_available()
        if device:
            return make_pattern_device(n, self.fa[interior], self.fb[interior], self.b if b is None else b,
                                       self.partition)
        a = self.fa[interior].astype(np.int64)
        c = self.fb[interior].astype(np.int64)
        rows = np.concatenate([np.arange(n), a, c])
        cols = np.concatenate([np.arange(n), c, a])
        key = np.unique(rows * n + cols)
        rows = (key // n).astype(np.int32)
        cols = (key % n).astype(np.int32)
        row_ptr = np.zeros(n + 1, np.int32)
        np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
        diag = np.flatnonzero(rows == cols).astype(np.int32)
        part = self.partition if self.partition is not None else np.zeros(n, np.int32)
        return dict(b=self.b if b is None else b, row_ptr=row_ptr, col_idx=cols, diag_idx=diag,
                    partition=np.ascontiguousarray(part, np.int32))

    def forcing_size(self):
        return 3 * self.n_boundary


def from_faces(n, fa, fb, fbc, ford, fn, vol, *, b=5, gamma=1.4, gas_constant=287.05, p0=101325.0, T0=300.0,
               p_out=98000.0, nt_in=0.0, forcing_scale=None, coords=None, mu=None, colour=None, partition=None,
               device=None):
    """Assemble the derived arrays (areas, unit normals, node->face CSR in ascending face
    order as mesh.cpp:44-59, slip-wall closure accumulated in face order) -- on the device
    (csrc/meshgen.cu, fnlh_mesh_derive) when one is present, else the host restatement."""
    fa = np.ascontiguousarray(fa, np.int32)
    fb = np.ascontiguousarray(fb, np.int32)
    fbc = np.ascontiguousarray(fbc, np.int32)
    ford = np.ascontiguousarray(ford, np.int32)
    fn = np.ascontiguousarray(np.asarray(fn, np.float64).reshape(-1, 3))
    nf = len(fa)
    interior = fbc < 0
    if device is None:
        device = _device_available()
    derive = _derive_device if device else _derive_host
    farea, fnh, fvis, nf_ptr, nf_idx, closure, bflag = derive(n, fa, np.where(interior, fb, -1).astype(np.int32), fn,
                                                              coords)
    m = Mesh3D(n=n, nf=nf, b=b, fa=fa, fb=fb, fbc=fbc, ford=ford, fn=fn.reshape(-1).copy(), farea=farea,
               fnh=np.ascontiguousarray(fnh.reshape(-1)), fvis=fvis, vol=np.ascontiguousarray(vol, np.float64),
               closure=closure.reshape(-1).copy(),
               mu=np.zeros(n) if mu is None else np.ascontiguousarray(mu, np.float64),
               nf_ptr=nf_ptr, nf_idx=nf_idx, bflag=bflag, gamma=gamma, gas_constant=gas_constant, p0=p0, T0=T0,
               p_out=p_out, nt_in=nt_in, forcing_scale=p_out if forcing_scale is None else forcing_scale,
               colour=None if colour is None else np.ascontiguousarray(colour, np.int32),
               partition=None if partition is None else np.ascontiguousarray(partition, np.int32),
               coords=coords, n_boundary=int((~interior).sum()))
    return m


def _derive_host(n, fa, fb, fn, coords):
    """Host restatement of fnlh_mesh_derive (mesh.cpp:44-59 + face/node derived arrays)."""
    nf = len(fa)
    farea = np.sqrt((fn[:, 0] * fn[:, 0] + fn[:, 1] * fn[:, 1]) + fn[:, 2] * fn[:, 2])
    fnh = fn / farea[:, None]
    interior = fb >= 0
    # node -> face CSR, ascending face index per node (Mesh::build_adjacency)
    ev_node = np.stack([fa, fb], axis=1).reshape(-1)
    ev_face = np.repeat(np.arange(nf, dtype=np.int32), 2)
    ev_sign = np.tile(np.array([1.0, -1.0]), nf)
    keep = ev_node >= 0
    ev_node, ev_face, ev_sign = ev_node[keep], ev_face[keep], ev_sign[keep]
    order = np.argsort(ev_node, kind="stable")  # events are in face order already
    nf_ptr = np.zeros(n + 1, np.int32)
    np.cumsum(np.bincount(ev_node, minlength=n), out=nf_ptr[1:])
    nf_idx = np.ascontiguousarray(ev_face[order], np.int32)
    # closure: start at 0.0 and add +-fn in face order per node (np.add.at is sequential)
    closure = np.zeros((n, 3))
    np.add.at(closure, ev_node, fn[ev_face] * ev_sign[:, None])
    bflag = np.zeros(n, np.int32)
    bflag[fa[~interior]] = 1
    fvis = np.zeros(nf)
    if coords is not None and interior.any():
        d = coords[fb[interior]] - coords[fa[interior]]
        fvis[interior] = farea[interior] / np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
    return farea, fnh, fvis, nf_ptr, nf_idx, closure, bflag


def _derive_device(n, fa, fb, fn, coords):
    import ctypes as C
    from ._lib import check, lib, ptr
    nf = len(fa)
    farea, fvis = np.empty(nf), np.empty(nf)
    fnh = np.empty((nf, 3))
    nf_ptr = np.empty(n + 1, np.int32)
    nf_idx = np.empty(2 * nf, np.int32)
    closure = np.empty((n, 3))
    bflag = np.empty(n, np.int32)
    X = None if coords is None else np.ascontiguousarray(coords, np.float64)
    check(lib().fnlh_mesh_derive(C.c_int(n), C.c_int(nf), ptr(np.ascontiguousarray(fa, np.int32)),
                                 ptr(np.ascontiguousarray(fb, np.int32)), ptr(np.ascontiguousarray(fn)), ptr(X),
                                 ptr(farea), ptr(fnh), ptr(fvis), ptr(nf_ptr), ptr(nf_idx), ptr(closure), ptr(bflag)))
    return farea, fnh, fvis, nf_ptr, np.ascontiguousarray(nf_idx[: nf_ptr[n]]), closure, bflag


def make_pattern_device(n, ea, eb, b=5, partition=None):
    """make_pattern (sparse.cpp:91-117) on the device (fnlh_make_pattern)."""
    import ctypes as C
    from ._lib import check, lib, ptr
    ea = np.ascontiguousarray(ea, np.int32)
    eb = np.ascontiguousarray(eb, np.int32)
    row_ptr = np.empty(n + 1, np.int32)
    col_idx = np.empty(n + 2 * len(ea), np.int32)
    diag = np.empty(n, np.int32)
    nnz = C.c_longlong()
    check(lib().fnlh_make_pattern(C.c_int(n), C.c_longlong(len(ea)), ptr(ea), ptr(eb), ptr(row_ptr), ptr(col_idx),
                                  ptr(diag), C.byref(nnz)))
    part = partition if partition is not None else np.zeros(n, np.int32)
    return dict(b=b, row_ptr=row_ptr, col_idx=np.ascontiguousarray(col_idx[: nnz.value]), diag_idx=diag,
                partition=np.ascontiguousarray(part, np.int32))


# ---------------------------------------------------------------------------- generators
def _cross(a, b):
    return np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1], a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
                     a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], axis=1)


_HEX_EDGES = [(p, p | (1 << d)) for d in range(3) for p in range(8) if not (p >> d) & 1]
_KUHN = [(0, 1 << a, (1 << a) | (1 << b), 7) for a, b, _ in itertools.permutations(range(3))]


def _hex_edge_faces(p, q):
    d = (p ^ q).bit_length() - 1
    faces = []
    for e in range(3):
        if e == d:
            continue
        bit = (p >> e) & 1
        faces.append([v for v in range(8) if ((v >> e) & 1) == bit])
    return faces


def _mean_cols(P, idx):
    """left-to-right sum of the listed corners / count (the device's order)"""
    acc = P[:, idx[0]].copy()
    for q in idx[1:]:
        acc = acc + P[:, q]
    return acc / float(len(idx))


def _dot3(a, b):
    return (a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1]) + a[:, 2] * b[:, 2]


def _tet_vol(a, b_, c, d):
    return np.abs(_dot3(b_ - a, _cross(c - a, d - a))) / 6.0


def _sector_cells(ci, cj, ck, periodic_j):
    nj_u, nk = cj + 1, ck + 1
    nj = cj if periodic_j else cj + 1
    ic, jc, kc = np.meshgrid(np.arange(ci), np.arange(cj), np.arange(ck), indexing="ij")
    ic, jc, kc = ic.reshape(-1), jc.reshape(-1), kc.reshape(-1)
    offs = [(c & 1, (c >> 1) & 1, (c >> 2) & 1) for c in range(8)]
    corners_u = np.stack([((ic + a) * nj_u + (jc + b)) * nk + (kc + c) for a, b, c in offs], axis=1)
    corners = np.stack([((ic + a) * nj + (jc + b) % nj) * nk + (kc + c) for a, b, c in offs], axis=1)
    return corners_u, corners


def _sector_dual_host(Xu, ci, cj, ck, periodic_j, tets):
    """Median-dual geometry of the structured sector (host restatement of csrc/meshgen.cu):
    per cell and edge the dual-face piece 0.5 (cen - m) x (c2 - c1) oriented along the edge,
    summed per edge in (template, cell) order; node volumes from the Kuhn tets.  Returns
    (ea, eb, en [ne, 3], vol [n]) with edges in ascending (ea, eb) order."""
    nj = cj if periodic_j else cj + 1
    n = (ci + 1) * nj * (ck + 1)
    corners_u, corners = _sector_cells(ci, cj, ck, periodic_j)
    P = Xu[corners_u]                                                # [ncell, 8, 3]
    e_keys, e_vecs = [], []
    vol_node = np.zeros(n)

    def add_edge(p_id, q_id, S, xp, xq):
        sgn = np.sign(_dot3(S, xq - xp))
        S = S * sgn[:, None]
        lo = np.minimum(p_id, q_id)
        hi = np.maximum(p_id, q_id)
        flip = np.where(p_id < q_id, 1.0, -1.0)
        e_keys.append(lo.astype(np.int64) * n + hi)
        e_vecs.append(S * flip[:, None])

    if not tets:
        cen = _mean_cols(P, list(range(8)))
        for (p, q) in _HEX_EDGES:
            f1, f2 = _hex_edge_faces(p, q)
            m = 0.5 * (P[:, p] + P[:, q])
            c1 = _mean_cols(P, f1)
            c2 = _mean_cols(P, f2)
            add_edge(corners[:, p], corners[:, q], 0.5 * _cross(cen - m, c2 - c1), P[:, p], P[:, q])
        vc = 0.0
        for t in _KUHN:
            vc = vc + _tet_vol(P[:, t[0]], P[:, t[1]], P[:, t[2]], P[:, t[3]])
        for c in range(8):
            vol_node += np.bincount(corners[:, c], weights=vc / 8.0, minlength=n)
    else:
        for t in _KUHN:
            T = P[:, list(t)]
            tid = corners[:, list(t)]
            cen = _mean_cols(T, [0, 1, 2, 3])
            vt = _tet_vol(T[:, 0], T[:, 1], T[:, 2], T[:, 3])
            for c in range(4):
                vol_node += np.bincount(tid[:, c], weights=vt / 4.0, minlength=n)
            for (p, q) in itertools.combinations(range(4), 2):
                r, s = [v for v in range(4) if v not in (p, q)]
                m = 0.5 * (T[:, p] + T[:, q])
                c1 = (T[:, p] + T[:, q] + T[:, r]) / 3.0
                c2 = (T[:, p] + T[:, q] + T[:, s]) / 3.0
                add_edge(tid[:, p], tid[:, q], 0.5 * _cross(cen - m, c2 - c1), T[:, p], T[:, q])
    keys = np.concatenate(e_keys)
    vecs = np.concatenate(e_vecs)
    ukeys, inv = np.unique(keys, return_inverse=True)
    en = np.stack([np.bincount(inv, weights=vecs[:, d], minlength=len(ukeys)) for d in range(3)], axis=1)
    return (ukeys // n).astype(np.int64), (ukeys % n).astype(np.int64), en, vol_node


def _device_available():
    try:
        from ._lib import lib
        return lib().fnlh_device_count() > 0
    except Exception:
        return False


def rcm_order(n, ea, eb, device=None):
    """Reverse Cuthill-McKee order of the graph with edges (ea, eb): rcm[position] = node.
    On the device (fnlh_rcm: level-synchronous BFS over the device-built pattern, equal to
    scipy's sequential algorithm) when one is present, else scipy.sparse.csgraph."""
    if device is None:
        device = _device_available()
    if device:
        from ._lib import check, lib, ptr
        pat = make_pattern_device(n, ea, eb)
        # component seeds exactly as scipy picks them: np.argsort of the int32 degrees
        # (numpy's default, unstable sort; the diagonal's +1 does not change the order)
        starts = np.ascontiguousarray(np.argsort(np.diff(pat["row_ptr"]).astype(np.int32)), np.int32)
        out = np.empty(n, np.int32)
        check(lib().fnlh_rcm(n, ptr(pat["row_ptr"]), ptr(pat["col_idx"]), ptr(starts), ptr(out)))
        return out.astype(np.int64)
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import reverse_cuthill_mckee
    ea = np.asarray(ea, np.int64)
    eb = np.asarray(eb, np.int64)
    G = coo_matrix((np.ones(2 * len(ea)), (np.concatenate([ea, eb]), np.concatenate([eb, ea]))), shape=(n, n)).tocsr()
    return np.asarray(reverse_cuthill_mckee(G, symmetric_mode=True), np.int64)


def graph_csr(n, ea, eb):
    """CSR adjacency + diagonal of the graph with edges (ea, eb): the host restatement of
    make_pattern's structure (sparse.cpp:91-117), rows with ascending unique columns."""
    a = np.asarray(ea, np.int64)
    c = np.asarray(eb, np.int64)
    rows = np.concatenate([np.arange(n), a, c])
    cols = np.concatenate([np.arange(n), c, a])
    key = np.unique(rows * n + cols)
    rows = (key // n).astype(np.int32)
    row_ptr = np.zeros(n + 1, np.int32)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return row_ptr, (key % n).astype(np.int32)


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def jp_priority(idx, seed):
    """Jones-Plassmann node priorities: splitmix64(seed + i * golden) high 32 bits above the
    node id (all distinct) -- meshgen.cu jp_priority, restated with wrapping uint64 math."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + np.asarray(idx, np.uint64) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return (z & np.uint64(0xFFFFFFFF00000000)) | np.asarray(idx, np.uint64)


def greedy_colouring(n, row_ptr, col_idx, seed=0x5EED, device=None):
    """Greedy colouring by Jones-Plassmann rounds: an uncoloured node whose priority beats
    every uncoloured neighbour's takes the smallest colour no coloured neighbour holds
    (colours of the previous round only).  On the device (fnlh_greedy_colour) when one is
    present; the host loop below is its exact restatement (the checker)."""
    if device is None:
        device = _device_available()
    rp = np.ascontiguousarray(row_ptr, np.int32)
    ci = np.ascontiguousarray(col_idx, np.int32)
    if device:
        import ctypes as C
        from ._lib import check, lib, ptr
        out = np.empty(n, np.int32)
        k = C.c_int()
        check(lib().fnlh_greedy_colour(C.c_int(n), ptr(rp), ptr(ci), C.c_ulonglong(seed), ptr(out), C.byref(k)))
        return out
    rows = np.repeat(np.arange(n), np.diff(rp))
    off = ci != rows
    rows, cols = rows[off], ci[off]
    prio = jp_priority(np.arange(n), seed)
    colour = np.full(n, -1, np.int64)
    while (colour < 0).any():
        unc = colour < 0
        # the largest priority among each node's uncoloured neighbours (0: none)
        nb_unc = unc[cols]
        best = np.zeros(n, np.uint64)
        np.maximum.at(best, rows[nb_unc], prio[cols[nb_unc]])
        used = np.zeros(n, np.uint64)
        col_nb = ~nb_unc
        np.bitwise_or.at(used, rows[col_nb], np.left_shift(np.uint64(1), colour[cols[col_nb]].astype(np.uint64)))
        top = unc & (prio > best)
        u = used[top]
        free = ~u & (u + np.uint64(1))  # lowest zero bit
        c = np.round(np.log2(free.astype(np.float64))).astype(np.int64)
        if (c >= 64).any() or (u == _M64).any():
            raise RuntimeError("greedy_colouring: more than 64 colours")
        colour[top] = c
    return colour.astype(np.int32)


def _sector_dual_device(Xu, ci, cj, ck, periodic_j, tets):
    """The same geometry from the sm_100a kernels (csrc/meshgen.cu, fnlh_sector_dual_*)."""
    import ctypes as C
    from ._lib import check, lib, ptr
    nj = cj if periodic_j else cj + 1
    n = (ci + 1) * nj * (ck + 1)
    X = np.ascontiguousarray(Xu, np.float64)
    h = C.c_void_p()
    ne = C.c_longlong()
    L = lib()
    check(L.fnlh_sector_dual_create(C.c_int(ci), C.c_int(cj), C.c_int(ck), C.c_int(int(periodic_j)),
                                    C.c_int(int(tets)), ptr(X), C.byref(ne), C.byref(h)))
    try:
        ea = np.empty(ne.value, np.int64)
        eb = np.empty(ne.value, np.int64)
        en = np.empty((ne.value, 3))
        vol = np.empty(n)
        check(L.fnlh_sector_dual_get(h, ptr(ea), ptr(eb), ptr(en), ptr(vol)))
    finally:
        L.fnlh_sector_dual_destroy(h)
    return ea, eb, en, vol


def morton_key(i, j, k) -> np.ndarray:
    """Z-order key of non-negative index triples (bits interleaved k, j, i from the top)."""
    key = np.zeros(len(i), np.int64)
    for bit in range(21):
        for t, v in enumerate((i, j, k)):
            key |= ((np.asarray(v, np.int64) >> bit) & 1) << (3 * bit + t)
    return key


def structured_sector(ci, cj, ck, *, geometry="annular", length=2.0, pitch_deg=10.0, r_in=0.5, r_out=1.0,
                      width=1.0, height=0.5, periodic_j=False, tets=False, jitter=0.0, seed=0, b=5, permute=True,
                      gas=None, nt_in=0.0, mu_range=None, device=None, order="rcm", colouring="structural"):
    """Hex (or Kuhn 6-tet) sector mesh, node-centred median dual.

    i: axial (inlet i=0, outlet i=ci), j: pitch, k: span/radius.  Walls (hub, casing,
    non-periodic pitch sides) enter through the closure source.  Returns a Mesh3D in
    colour-major RCM order (2 colours for hex, 8 for Kuhn tets).

    order: the node numbering inside each colour -- "rcm" (seeded permutation, then reverse
    Cuthill-McKee), "lex" / "lexk" (lexicographic in the index triple) or "morton" (Z-order of the (i, j, k) index triple: a cache-oblivious
    renumbering for locality, so the neighbours a row gathers were touched recently by the
    rows around it).  On a 2-colour ordering the ILU(0) entries do not depend on the order
    inside a colour (only the summation order of each row's Schur update does).

    colouring: "structural" ((i+j+k) mod 2 for hex, the 8 Kuhn colours for tets) or "greedy":
    the Jones-Plassmann colouring of the seeded-permuted node graph (greedy_colouring), as a
    mesh without structured indices gets -- then colour-major with RCM inside each colour.

    device: compute the dual geometry (per-cell dual-face normals, their per-edge sums,
    node volumes) with the sm_100a kernels of csrc/meshgen.cu (bitwise equal to the host
    restatement `_sector_dual_host`); None = on the device when one is present."""
    if device is None:
        device = _device_available()
    rng = np.random.default_rng(seed)
    ni, nj_u, nk = ci + 1, cj + 1, ck + 1
    nj = cj if periodic_j else cj + 1
    I, J, K = np.meshgrid(np.arange(ni), np.arange(nj_u), np.arange(nk), indexing="ij")
    fi, fj, fk = I.astype(float), J.astype(float), K.astype(float)
    if jitter > 0.0:
        inner = (I > 0) & (I < ci) & (J > 0) & (J < cj) & (K > 0) & (K < ck)
        jit = rng.uniform(-jitter, jitter, size=(3,) + I.shape)
        fi = fi + np.where(inner, jit[0], 0.0)
        fj = fj + np.where(inner, jit[1], 0.0)
        fk = fk + np.where(inner, jit[2], 0.0)
    if geometry == "annular":
        th = np.deg2rad(pitch_deg) * fj / cj
        r = r_in + (r_out - r_in) * fk / ck
        X = np.stack([length * fi / ci, r * np.cos(th), r * np.sin(th)], axis=-1)
    else:
        X = np.stack([length * fi / ci, width * fj / cj, height * fk / ck], axis=-1)
    Xu = X.reshape(-1, 3)                                            # unwrapped coordinates
    gid = ((I * nj + (J % nj)) * nk + K).reshape(-1)                 # mapped node id
    n = ni * nj * nk
    coords = np.ascontiguousarray(X[:, :nj, :].reshape(-1, 3))     # gid order (seam copies dropped)
    uid = lambda i, j, k: (i * nj_u + j) * nk + k  # noqa: E731
    # hex cells: corner c = di + 2 dj + 4 dk
    if device:
        ea, eb, en, vol_node = _sector_dual_device(Xu, ci, cj, ck, periodic_j, tets)
    else:
        ea, eb, en, vol_node = _sector_dual_host(Xu, ci, cj, ck, periodic_j, tets)

    # inlet (i=0, outward -x) and outlet (i=ci, outward +x) dual boundary areas
    jq, kq = np.meshgrid(np.arange(cj), np.arange(ck), indexing="ij")
    jq, kq = jq.reshape(-1), kq.reshape(-1)
    b_nodes, b_vecs, b_kind = [], [], []
    for kind, iplane, out in ((0, 0, -1.0), (1, ci, 1.0)):
        q_u = np.stack([uid(iplane, jq, kq), uid(iplane, jq + 1, kq), uid(iplane, jq + 1, kq + 1),
                        uid(iplane, jq, kq + 1)], axis=1)
        Q = Xu[q_u]
        polys = [[0, 1, 2], [0, 2, 3]] if tets else [[0, 1, 2, 3]]
        acc = np.zeros(n)
        for poly in polys:
            V = Q[:, poly]
            cen = V.mean(axis=1)
            L = len(poly)
            for t in range(L):
                p, nx_, pv = V[:, t], V[:, (t + 1) % L], V[:, (t - 1) % L]
                S = 0.5 * _cross(cen - p, 0.5 * (p + pv) - 0.5 * (p + nx_))
                acc += np.bincount(gid[q_u[:, poly[t]]], weights=np.abs(S[:, 0]), minlength=n)
        nodes = np.flatnonzero(acc > 0)
        b_nodes.append(nodes)
        b_vecs.append(np.stack([out * acc[nodes], np.zeros(len(nodes)), np.zeros(len(nodes))], axis=1))
        b_kind.append(np.full(len(nodes), kind))
    b_nodes = np.concatenate(b_nodes)
    b_vecs = np.concatenate(b_vecs)
    b_kind = np.concatenate(b_kind)

    # structural colouring: 2 colours (hex, (i+j+k) mod 2), 8 colours (Kuhn tets)
    In, Jn, Kn = np.meshgrid(np.arange(ni), np.arange(nj), np.arange(nk), indexing="ij")
    col = ((In + Jn + Kn) % 2) if not tets else ((In + 2 * Jn + 4 * Kn) % 8)
    col = col.reshape(-1).astype(np.int32)
    if periodic_j and not tets:
        assert cj % 2 == 0, "periodic 2-colouring needs an even pitch count"

    # ordering: seeded permutation -> RCM (or Morton) -> colour-major (stable)
    perm0 = rng.permutation(n) if permute else np.arange(n)        # perm0[new] = old
    if colouring == "greedy":  # colours of the permuted graph, as an unstructured mesh has them
        inv_p = np.empty(n, np.int64)
        inv_p[perm0] = np.arange(n)
        rp_, ci_ = graph_csr(n, inv_p[ea], inv_p[eb])
        col = greedy_colouring(n, rp_, ci_, seed=seed + 1, device=device)[inv_p].astype(np.int32)
    elif colouring != "structural":
        raise ValueError(f"unknown colouring {colouring!r}")
    if order == "morton":
        rank = morton_key(In.reshape(-1), Jn.reshape(-1), Kn.reshape(-1))  # rank[old], gid order
    elif order in ("lex", "lexk"):
        # lexicographic index order: every neighbour slot of 32 consecutive rows is one
        # contiguous run of nodes ("lex": i fastest; "lexk": k fastest)
        I_, J_, K_ = (a.reshape(-1).astype(np.int64) for a in (In, Jn, Kn))
        mi, mj, mk = int(I_.max()) + 1, int(J_.max()) + 1, int(K_.max()) + 1
        rank = (K_ * mj + J_) * mi + I_ if order == "lex" else (I_ * mj + J_) * mk + K_
    elif order == "rcm":
        inv0 = np.empty(n, np.int64)
        inv0[perm0] = np.arange(n)
        ra, rb = inv0[ea], inv0[eb]
        rcm = rcm_order(n, ra, rb, device)                           # rcm[pos] = permuted id
        rank = np.empty(n, np.int64)
        rank[perm0[rcm]] = np.arange(n)                              # rank[old] = RCM position
    else:
        raise ValueError(f"unknown node order {order!r}")
    order = np.lexsort((rank, col))                                  # order[new] = old
    new = np.empty(n, np.int64)
    new[order] = np.arange(n)

    a2, b2 = new[ea], new[eb]
    sw = a2 > b2
    en = np.where(sw[:, None], -en, en)
    a2, b2 = np.where(sw, b2, a2), np.where(sw, a2, b2)
    o = np.lexsort((b2, a2))
    a2, b2, en = a2[o], b2[o], en[o]
    bn = new[b_nodes]
    ob = np.lexsort((bn, b_kind))
    bn, b_vecs, b_kind = bn[ob], b_vecs[ob], b_kind[ob]
    ne, nb = len(a2), len(bn)
    fa = np.concatenate([a2, bn]).astype(np.int32)
    fb = np.concatenate([b2, -np.ones(nb, np.int64)]).astype(np.int32)
    fbc = np.concatenate([-np.ones(ne, np.int64), b_kind]).astype(np.int32)
    ford = np.concatenate([np.zeros(ne, np.int64), np.arange(nb)]).astype(np.int32)
    fnv = np.concatenate([en, b_vecs])
    g = gas or {}
    mu = None
    if mu_range is not None:
        lo_, hi_ = np.log(mu_range[0]), np.log(mu_range[1])
        mu = np.exp(rng.uniform(lo_, hi_, size=n))
    m = from_faces(n, fa, fb, fbc, ford, fnv, vol_node[order], b=b, coords=coords[order], colour=col[order],
                   mu=mu, nt_in=nt_in, device=device, **g)
    m.ijk = np.stack([In.reshape(-1), Jn.reshape(-1), Kn.reshape(-1)], axis=1)[order].astype(np.int64)
    return m


# ---------------------------------------------------------------------------- multigrid
def parent_map(ijk) -> np.ndarray:
    """fine node -> coarse node of the 2x2x2 agglomeration of structured nodes (the 3D
    counterpart of multigrid.cpp:9-24: pairwise in 1D, 2x2 in 2D).  Coarse nodes are
    numbered in lexicographic (i, j, k) order of their index triple, so a line mesh gets the
    reference's parent[i] = i / 2."""
    c = np.asarray(ijk, np.int64) // 2
    dims = c.max(axis=0) + 1
    key = (c[:, 0] * dims[1] + c[:, 1]) * dims[2] + c[:, 2]
    _, parent = np.unique(key, return_inverse=True)
    return parent.astype(np.int32)


def coarsen(m: Mesh3D, parent, forcing=None):
    """Agglomerated coarse mesh (multigrid.cpp:41-127 restated for median-dual faces).

    * coarse volume = child volumes summed in ascending fine order; coarse position and
      eddy viscosity volume-weighted;
    * coarse interior face between agglomerates P < Q = the fine faces crossing from P to
      Q, normals summed in fine face order (one fine face per coarse face on a line mesh:
      the reference's "areas transfer unchanged");
    * coarse boundary face per (boundary kind, agglomerate), normals summed; its forcing
      slot is the area-weighted mean of the children's (copied when there is one child);
    * walls stay implicit: the closure is rebuilt from the coarse faces (from_faces).

    Returns (coarse mesh, coarse forcing [nh, 3 * n_boundary] or None)."""
    parent = np.asarray(parent, np.int64)
    nc = int(parent.max()) + 1
    vol = np.zeros(nc)
    np.add.at(vol, parent, m.vol)
    fn = m.fn.reshape(-1, 3)
    interior = m.fbc < 0
    P, Q, nrm = parent[m.fa[interior]], parent[m.fb[interior]], fn[interior]
    keep = P != Q
    P, Q, nrm = P[keep], Q[keep], nrm[keep]
    sw = P > Q
    P, Q = np.where(sw, Q, P), np.where(sw, P, Q)
    nrm = np.where(sw[:, None], -nrm, nrm)
    key = P * nc + Q
    ukey, inv = np.unique(key, return_inverse=True)
    cfn = np.zeros((len(ukey), 3))
    np.add.at(cfn, inv, nrm)
    live = np.any(cfn != 0.0, axis=1)  # a periodic pair of agglomerates can cancel exactly
    ukey, cfn = ukey[live], cfn[live]
    ca, cb = (ukey // nc).astype(np.int32), (ukey % nc).astype(np.int32)
    # boundary faces, grouped per (kind, agglomerate)
    bidx = np.flatnonzero(~interior)
    bk, bp = m.fbc[bidx].astype(np.int64), parent[m.fa[bidx]]
    bkey = bk * nc + bp
    ubkey, binv = np.unique(bkey, return_inverse=True)
    bfn = np.zeros((len(ubkey), 3))
    np.add.at(bfn, binv, fn[bidx])
    nbc = len(ubkey)
    fa = np.concatenate([ca, (ubkey % nc).astype(np.int32)])
    fb = np.concatenate([cb, -np.ones(nbc, np.int32)])
    fbc = np.concatenate([-np.ones(len(ca), np.int32), (ubkey // nc).astype(np.int32)])
    ford = np.concatenate([np.zeros(len(ca), np.int32), np.arange(nbc, dtype=np.int32)])
    coords = None
    if m.coords is not None:
        coords = np.zeros((nc, 3))
        np.add.at(coords, parent, m.coords * m.vol[:, None])
        coords /= vol[:, None]
    mu = np.zeros(nc)
    np.add.at(mu, parent, m.mu * m.vol)
    mu /= vol
    c = from_faces(nc, fa, fb, fbc, ford, np.concatenate([cfn, bfn]), vol, b=m.b, gamma=m.gamma,
                   gas_constant=m.gas_constant, p0=m.p0, T0=m.T0, p_out=m.p_out, nt_in=m.nt_in,
                   forcing_scale=m.forcing_scale, coords=coords, mu=mu)
    if m.ijk is not None:
        ijk = np.zeros((nc, 3), np.int64)
        ijk[parent] = np.asarray(m.ijk, np.int64) // 2
        c.ijk = ijk
    cf = None
    if forcing is not None:
        fz = np.asarray(forcing, np.complex128).reshape(len(forcing), -1, 3)  # [nh, n_boundary, 3]
        ordv = m.ford[bidx]
        area = m.farea[bidx]
        cnt = np.bincount(binv, minlength=nbc)
        num = np.zeros((fz.shape[0], nbc, 3), np.complex128)
        den = np.zeros(nbc)
        np.add.at(den, binv, area)
        for h in range(fz.shape[0]):
            np.add.at(num[h], binv, fz[h][ordv] * area[:, None])
        cf = num / den[None, :, None]
        single = np.flatnonzero(cnt == 1)
        if len(single):
            first = np.zeros(nbc, np.int64)
            first[binv[::-1]] = np.arange(len(binv))[::-1]
            cf[:, single, :] = fz[:, ordv[first[single]], :]
        cf = cf.reshape(fz.shape[0], -1)
    return c, cf


def hierarchy(m: Mesh3D, levels: int, forcing=None):
    """build_hierarchy (multigrid.cpp:129-140): [(mesh, parent-into-next, forcing)] per
    level, finest first (parent is None on the coarsest)."""
    if levels < 1:
        raise ValueError("hierarchy needs at least one level")
    if levels > 1 and m.ijk is None:
        raise ValueError("coarsening needs structured node indices (Mesh3D.ijk)")
    out = []
    cur, cf = m, forcing
    for lv in range(levels):
        if lv + 1 < levels:
            par = parent_map(cur.ijk)
            nxt, nf = coarsen(cur, par, cf)
            out.append((cur, par, cf))
            cur, cf = nxt, nf
        else:
            out.append((cur, None, cf))
    return out
