"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU checkers.

* ``Oracle``  -> oracle/liboracle.so, the plain-C restatement (fnlh_oracle.c).
* ``RefLib``  -> oracle/_ref/libfnlh_ref.so, the UNMODIFIED reference compiled from
  /root/reference/proj/src + ref_bridge.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfnlh_ref.so")

_i = C.c_int
_d = C.c_double
_p = C.c_void_p

ERR_NAMES = {1: "ConfigError", 2: "StateError", 3: "ShapeError", 4: "UnsupportedCaseError",
             5: "FactorizationError", 6: "DivergenceError", 99: "std::exception"}


class CheckerError(RuntimeError):
    def __init__(self, code, msg, node=-1, stage=-1):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code, self.node, self.stage = code, node, stage


def ptr(a):
    return None if a is None else a.ctypes.data_as(_p)


def build(quiet=True):
    """Compile the restatement (and the reference bridge where /root/reference exists)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def ref_available():
    return os.path.exists(REF_SO)


# --------------------------------------------------------------------------- structs
class OrPattern(C.Structure):
    _fields_ = [("b", _i), ("rows", _i), ("nnzb", _i), ("row_ptr", _p), ("col_idx", _p),
                ("diag_idx", _p), ("partition", _p)]


class OrIlu(C.Structure):
    _fields_ = [("vals", _p), ("diag_lu", _p), ("diag_piv", _p), ("diag_inv", _p)]


class OrReport(C.Structure):
    _fields_ = [("iterations", _i), ("initial_residual", _d), ("final_residual", _d), ("converged", _i)]


class OrMesh(C.Structure):
    _fields_ = [("n", _i), ("nf", _i), ("b", _i), ("fa", _p), ("fb", _p), ("fbc", _p), ("ford", _p),
                ("fn", _p), ("farea", _p), ("fnh", _p), ("fvis", _p), ("vol", _p), ("closure", _p),
                ("mu", _p), ("nf_ptr", _p), ("nf_idx", _p), ("bflag", _p), ("gamma", _d),
                ("gas_constant", _d), ("p0", _d), ("T0", _d), ("p_out", _d), ("nt_in", _d),
                ("forcing_scale", _d)]


class OrScheme(C.Structure):
    _fields_ = [("implicit", _i), ("sigma_cfl", _d), ("eps_relax", _d), ("linear_tol", _d),
                ("linear_max_iter", _i), ("target_drop_orders", _d), ("max_outer_iters", _i)]


class OrEntry(C.Structure):
    _fields_ = [("iter", _i), ("resid_mean", _d), ("rz", _d), ("has_rz", _i), ("stage1_norm_mean", _d)]


class OrError(C.Structure):
    _fields_ = [("code", _i), ("node", _i), ("stage", _i), ("msg", C.c_char * 256)]


# --------------------------------------------------------------------------- restatement
class Oracle:
    """The plain-C restatement (liboracle.so)."""

    def __init__(self, path=ORACLE_SO, pow_mode="glibc", workers=1):
        """pow_mode: "glibc" evaluates the boundary-state pow with the reference's libm,
        "cr" with the device's correctly rounded pow (oracle/cr_pow.h).  workers: harmonic
        worker threads (SchemeConfig::workers, driver.cpp:246-265)."""
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        self.cr = 1 if pow_mode == "cr" else 0
        self.workers = int(workers)
        L.or_last_error.restype = C.POINTER(OrError)
        L.or_solver_create.restype = _p
        L.or_solver_df.restype = C.POINTER(_d)
        self._keep = []

    def mode(self):
        self.lib.or_set_pow_mode(_i(self.cr))
        self.lib.or_set_workers(_i(self.workers))
        return self.lib

    def _check(self, st):
        if st:
            e = self.lib.or_last_error().contents
            raise CheckerError(e.code, e.msg.decode(), e.node, e.stage)

    # -- pattern / mesh plumbing
    def pattern(self, pat):
        """pat: dict with b, row_ptr, col_idx, diag_idx, partition (int32 arrays)."""
        keep = [pat["row_ptr"], pat["col_idx"], pat["diag_idx"], pat["partition"]]
        self._keep.append(keep)
        return OrPattern(int(pat["b"]), len(pat["row_ptr"]) - 1, len(pat["col_idx"]), ptr(keep[0]),
                         ptr(keep[1]), ptr(keep[2]), ptr(keep[3]))

    def mesh(self, m):
        """m: paper_2404_01407_b200.mesh.Mesh3D (or any object with the same fields)."""
        keep = [m.fa, m.fb, m.fbc, m.ford, m.fn, m.farea, m.fnh, m.fvis, m.vol, m.closure, m.mu,
                m.nf_ptr, m.nf_idx, m.bflag]
        self._keep.append(keep)
        return OrMesh(m.n, m.nf, m.b, *[ptr(a) for a in keep], m.gamma, m.gas_constant, m.p0, m.T0,
                      m.p_out, m.nt_in, m.forcing_scale)

    # -- LA
    def ilu_factorize(self, pat, A):
        cplx = np.iscomplexobj(A)
        b, n = pat["b"], len(pat["row_ptr"]) - 1
        dt = np.complex128 if cplx else np.float64
        vals = np.zeros_like(A, dtype=dt)
        dlu = np.zeros(n * b * b, dt)
        piv = np.zeros(n * b, np.int32)
        dinv = np.zeros(n * b * b, dt)
        P = self.pattern(pat)
        f = OrIlu(ptr(vals), ptr(dlu), ptr(piv), ptr(dinv))
        A = np.ascontiguousarray(A, dtype=dt)
        fn = self.mode().or_ilu_factorize_z if cplx else self.lib.or_ilu_factorize_d
        self._check(fn(C.byref(P), ptr(A), C.byref(f)))
        return dict(vals=vals, diag_lu=dlu, diag_piv=piv, diag_inv=dinv)

    def smoothed_solve(self, pat, A, rhs, tol, max_iter):
        cplx = np.iscomplexobj(A)
        dt = np.complex128 if cplx else np.float64
        ilu = self.ilu_factorize(pat, A)
        P = self.pattern(pat)
        f = OrIlu(ptr(ilu["vals"]), ptr(ilu["diag_lu"]), ptr(ilu["diag_piv"]), ptr(ilu["diag_inv"]))
        x = np.zeros(len(rhs), dt)
        rep = OrReport()
        A = np.ascontiguousarray(A, dtype=dt)
        rhs = np.ascontiguousarray(rhs, dtype=dt)
        fn = self.lib.or_smoothed_solve_z if cplx else self.lib.or_smoothed_solve_d
        self._check(fn(C.byref(P), ptr(A), ptr(rhs), C.byref(f), _d(tol), _i(max_iter), ptr(x), C.byref(rep)))
        return x, (rep.iterations, rep.initial_residual, rep.final_residual, bool(rep.converged))

    # -- full-size harmonic workers (bench.py --impl reference): the reference's own objects
    def lhs_create(self, pat, A5):
        """The shared real LHS A5 on its pattern (Bsr<real>); keep the handle alive while
        workers use it."""
        self._lhs_keep = [np.ascontiguousarray(pat["row_ptr"]), np.ascontiguousarray(pat["col_idx"]),
                          np.ascontiguousarray(A5, np.float64)]
        b, n = int(pat["b"]), len(pat["row_ptr"]) - 1
        self.lib.ref_lhs_create.restype = _p
        h = self.lib.ref_lhs_create(_i(b), _i(n), ptr(self._lhs_keep[0]), ptr(self._lhs_keep[1]), ptr(self._lhs_keep[2]))
        if not h:
            self._check(7)
        return h

    def hworker_create(self, lhs, shift_im, rhs):
        """One harmonic worker: shift_diagonal into its complex workspace + Ilu factorize.
        Returns (handle, factorization seconds)."""
        fs = _d()
        self.lib.ref_hworker_create.restype = _p
        sh = np.ascontiguousarray(shift_im, np.float64)
        r = np.ascontiguousarray(rhs, np.complex128)
        h = self.lib.ref_hworker_create(_p(lhs), ptr(sh), ptr(r), C.byref(fs))
        if not h:
            self._check(7)
        return h, fs.value

    def hworker_sweeps(self, w, sweeps):
        """smoothed_solve of `sweeps` iterations on the worker's system: (seconds, final norm)."""
        t, f = _d(), _d()
        self._check(self.lib.ref_hworker_sweeps(_p(w), _i(sweeps), C.byref(t), C.byref(f)))
        return t.value, f.value

    def hworker_destroy(self, w):
        self.lib.ref_hworker_destroy(_p(w))

    def lhs_destroy(self, h):
        self.lib.ref_lhs_destroy(_p(h))

    def build_lhs_mean(self, pat, J, implicit, sigma, eps, stage):
        A = np.zeros_like(J)
        P = self.pattern(pat)
        self._check(self.mode().or_build_lhs_mean(C.byref(P), ptr(J), _i(implicit), _d(sigma), _d(eps), _i(stage),
                                               ptr(A)))
        return A

    # -- discretization
    def residual(self, m, W, order, mode=0, wref=None, forcing=None, need_vis=False):
        M = self.mesh(m)
        n = m.n * m.b
        inv = np.zeros(n)
        vis = np.zeros(n)
        f = None if forcing is None else np.ascontiguousarray(forcing, np.float64)
        self._check(self.mode().or_residual(C.byref(M), ptr(np.ascontiguousarray(W)), ptr(wref), _i(order), _i(mode),
                                         ptr(f), _i(0 if f is None else len(f)), _i(int(need_vis)), ptr(inv),
                                         ptr(vis)))
        return inv, vis

    def fd_jacobian(self, m, pat, W, want_J=True, want_P=False):
        M = self.mesh(m)
        P = self.pattern(pat)
        b = m.b
        J = np.zeros(len(pat["col_idx"]) * b * b) if want_J else None
        D = np.zeros(m.n * b * b) if want_P else None
        self._check(self.mode().or_fd_jacobian(C.byref(M), C.byref(P), ptr(np.ascontiguousarray(W)), ptr(J), ptr(D)))
        return J, D

    def transform_jacobian(self, m, W):
        out = np.zeros(m.n * m.b * m.b)
        self._check(self.mode().or_transform_jacobian(_i(m.b), _i(m.n), _d(m.gamma), ptr(np.ascontiguousarray(W)),
                                                   ptr(out)))
        return out

    def linearized_residual(self, m, mean, what, omega, forcing, order=2, need_vis=True):
        Mm = self.mesh(m)
        M = self.transform_jacobian(m, mean)
        n = m.n * m.b
        inv = np.zeros(n, np.complex128)
        vis = np.zeros(n, np.complex128)
        f = np.ascontiguousarray(forcing, np.complex128)
        self._check(self.mode().or_linearized_residual(C.byref(Mm), ptr(np.ascontiguousarray(mean)), ptr(M),
                                                    ptr(np.ascontiguousarray(what, np.complex128)), _d(omega),
                                                    ptr(f), _i(len(f)), _i(order), _i(int(need_vis)), ptr(inv),
                                                    ptr(vis)))
        return inv, vis

    def deterministic_flux(self, m, mean, omegas, amps, index=None):
        Mm = self.mesh(m)
        nh = len(omegas)
        idx = np.arange(1, nh + 1, dtype=np.int32) if index is None else np.asarray(index, np.int32)
        om = np.asarray(omegas, np.float64)
        a = np.ascontiguousarray(amps, np.complex128)
        df = np.zeros(m.n * m.b)
        self._check(self.mode().or_deterministic_flux(C.byref(Mm), ptr(np.ascontiguousarray(mean)), _i(nh), ptr(idx),
                                                   ptr(om), ptr(a), ptr(df)))
        return df

    # -- solver
    def solver(self, m, pat, scheme, omegas, forcing, mean0, index=None):
        return OracleSolver(self, m, pat, scheme, omegas, forcing, mean0, index)


class OracleSolver:
    def __init__(self, orc, m, pat, scheme, omegas, forcing, mean0, index=None):
        self.o = orc
        self.m = m
        self.nh = len(omegas)
        self.Mm = orc.mesh(m)
        self.P = orc.pattern(pat)
        self.S = OrScheme(int(scheme.get("implicit", 1)), scheme.get("sigma_cfl", -1.0), scheme.get("eps_relax", 0.6),
                          scheme.get("linear_tol", 1e-2), scheme.get("linear_max_iter", 10),
                          scheme.get("target_drop_orders", 8.0), scheme.get("max_outer_iters", 2000))
        idx = np.arange(1, self.nh + 1, dtype=np.int32) if index is None else np.asarray(index, np.int32)
        self._keep = [idx, np.asarray(omegas, np.float64), np.ascontiguousarray(forcing, np.complex128),
                      np.ascontiguousarray(mean0, np.float64)]
        nf = self._keep[2].shape[-1] if self.nh else 0
        self.h = orc.lib.or_solver_create(C.byref(self.Mm), C.byref(self.P), C.byref(self.S), _i(self.nh),
                                          ptr(self._keep[0]), ptr(self._keep[1]), ptr(self._keep[2]), _i(nf),
                                          ptr(self._keep[3]))
        levels = int(scheme.get("mg_levels", 1))
        if levels > 1:  # the same 2x2x2 hierarchy the device solver builds
            from paper_2404_01407_b200.mesh import hierarchy
            hier = hierarchy(m, levels, self._keep[2] if self.nh else None)
            for lv in range(1, levels):
                self.add_level(hier[lv][0], hier[lv - 1][1], hier[lv][2])

    def __del__(self):
        try:
            self.o.lib.or_solver_destroy(_p(self.h))
        except Exception:
            pass

    def add_level(self, m, parent, forcing=None):
        """Append a coarse multigrid level (explicit scheme): Mesh3D m, parent map from the
        current coarsest level's nodes, the level's boundary forcing [nh, nforcing]."""
        pat = m.pattern()
        Mm = self.o.mesh(m)
        P = self.o.pattern(pat)
        par = np.ascontiguousarray(parent, np.int32)
        fz = np.ascontiguousarray(forcing if forcing is not None else np.zeros((self.nh, 0)), np.complex128)
        nf = fz.shape[-1] if self.nh else 0
        self._keep += [Mm, P, pat, par, fz]
        self.o._check(self.o.lib.or_solver_add_level(_p(self.h), C.byref(Mm), C.byref(P), ptr(par), ptr(fz), _i(nf)))

    def outer_iteration(self):
        e = OrEntry()
        rh = np.zeros(max(self.nh, 1))
        self.o._check(self.o.mode().or_solver_outer_iteration(_p(self.h), C.byref(e), ptr(rh)))
        return dict(iter=e.iter, resid_mean=e.resid_mean, rz=e.rz, has_rz=bool(e.has_rz),
                    resid_h=rh[: self.nh].copy(), stage1_norm_mean=e.stage1_norm_mean)

    # the two halves of outer_iteration (harmonic sharding)
    def phase_harmonics(self, owned=None):
        hn = np.zeros(max(self.nh, 1))
        own = None if owned is None else np.ascontiguousarray(owned, np.int32)
        self.o._check(self.o.mode().or_solver_phase_harmonics(_p(self.h), ptr(own), ptr(hn)))
        return hn[: self.nh].copy()

    def failed_harmonic(self):
        return self.o.lib.or_solver_failed_harmonic(_p(self.h))

    # deterministic_flux split over quadrature points (host pointers)
    def df_points(self):
        return self.o.lib.or_solver_df_points(_p(self.h))

    def df_terms(self, k0, k1, terms_ptr):
        self.o._check(self.o.lib.or_solver_df_terms(_p(self.h), _i(k0), _i(k1), _p(terms_ptr)))

    def df_accumulate(self, terms_ptr, count, acc_ptr, first):
        self.o.lib.or_solver_df_accumulate(_p(self.h), _p(terms_ptr), _i(count), _p(acc_ptr), _i(1 if first else 0))

    def set_external_df(self, acc_ptr):
        self.o.lib.or_solver_set_external_df(_p(self.h), _p(acc_ptr))

    def harmonic_reports(self, h):
        arr = (OrReport * 256)()
        k = self.o.lib.or_solver_harmonic_reports(_p(self.h), _i(h), arr, _i(256))
        return [(r.iterations, r.initial_residual, r.final_residual, bool(r.converged)) for r in arr[:k]]

    def phase_mean(self, h_norm, h_reports):
        reps = [r for hr in h_reports for r in hr]
        arr = (OrReport * max(len(reps), 1))(*[OrReport(r[0], r[1], r[2], int(r[3])) for r in reps])
        nrep = np.array([len(hr) for hr in h_reports] + [0], np.int32)
        e = OrEntry()
        rh = np.zeros(max(self.nh, 1))
        self.o._check(self.o.mode().or_solver_phase_mean(_p(self.h), ptr(np.ascontiguousarray(h_norm, np.float64)),
                                                          ptr(nrep), arr, C.byref(e), ptr(rh)))
        return dict(iter=e.iter, resid_mean=e.resid_mean, rz=e.rz, has_rz=bool(e.has_rz),
                    resid_h=rh[: self.nh].copy(), stage1_norm_mean=e.stage1_norm_mean)

    def get_amps(self, h):
        return self.state()[1][h]

    def put_amps(self, h, a):
        mean, amps = self.state()
        amps[h] = a
        self.set_state(mean, amps)

    def state(self):
        n = self.m.n * self.m.b
        mean = np.zeros(n)
        amps = np.zeros(self.nh * n, np.complex128)
        self.o.lib.or_solver_get_state(_p(self.h), ptr(mean), ptr(amps))
        return mean, amps.reshape(self.nh, n)

    def set_state(self, mean, amps):
        self.o.lib.or_solver_set_state(_p(self.h), ptr(np.ascontiguousarray(mean, np.float64)),
                                       ptr(np.ascontiguousarray(amps, np.complex128)))

    def df(self):
        n = self.m.n * self.m.b
        return np.ctypeslib.as_array(self.o.lib.or_solver_df(_p(self.h)), shape=(n,)).copy()

    def reports(self):
        k = self.o.lib.or_solver_num_reports(_p(self.h))
        arr = (OrReport * max(k, 1))()
        self.o.lib.or_solver_get_reports(_p(self.h), arr)
        return [(r.iterations, r.initial_residual, r.final_residual, bool(r.converged)) for r in arr[:k]]


# --------------------------------------------------------------------------- reference
class RefLib:
    """The reference itself (oracle/_ref/libfnlh_ref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path + " (build with `make -C oracle` where /root/reference exists)")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_nozzle_create.restype = _p
        L.ref_solver_create.restype = _p
        L.ref_time_sweeps_d.restype = _d
        L.ref_time_sweeps_z.restype = _d

    def _check(self, st):
        if st:
            raise CheckerError(st, self.lib.ref_last_error().decode(), self.lib.ref_last_error_node(),
                               self.lib.ref_last_error_stage())

    @staticmethod
    def _csr(pat):
        part = pat.get("partition")
        return (int(pat["b"]), len(pat["row_ptr"]) - 1, ptr(pat["row_ptr"]), ptr(pat["col_idx"]),
                None if part is None else ptr(part))

    def make_pattern(self, b, rows, ea, eb):
        """The reference's make_pattern (sparse.cpp:91-117) on an edge list."""
        ea = np.ascontiguousarray(ea, np.int32)
        eb = np.ascontiguousarray(eb, np.int32)
        row_ptr = np.empty(rows + 1, np.int32)
        col_idx = np.empty(rows + 2 * len(ea), np.int32)
        diag = np.empty(rows, np.int32)
        nnz = C.c_longlong()
        self._check(self.lib.ref_make_pattern(_i(b), _i(rows), C.c_longlong(len(ea)), ptr(ea), ptr(eb), ptr(row_ptr),
                                              ptr(col_idx), ptr(diag), C.byref(nnz)))
        return dict(row_ptr=row_ptr, col_idx=col_idx[: nnz.value].copy(), diag_idx=diag)

    def build_adjacency(self, n, fa, fb):
        """Mesh::build_adjacency (mesh.cpp:44-59) on a face list (fb = -1 on boundary faces)."""
        fa = np.ascontiguousarray(fa, np.int32)
        fb = np.ascontiguousarray(fb, np.int32)
        nf_ptr = np.empty(n + 1, np.int32)
        nf_idx = np.empty(2 * len(fa), np.int32)
        self._check(self.lib.ref_build_adjacency(_i(n), _i(len(fa)), ptr(fa), ptr(fb), ptr(nf_ptr), ptr(nf_idx)))
        return nf_ptr, nf_idx[: nf_ptr[n]].copy()

    def ilu_factorize(self, pat, A):
        cplx = np.iscomplexobj(A)
        dt = np.complex128 if cplx else np.float64
        b, n = pat["b"], len(pat["row_ptr"]) - 1
        A = np.ascontiguousarray(A, dt)
        vals = np.zeros_like(A)
        dlu = np.zeros(n * b * b, dt)
        piv = np.zeros(n * b, np.int32)
        dinv = np.zeros(n * b * b, dt)
        fn = self.lib.ref_ilu_factorize_z if cplx else self.lib.ref_ilu_factorize_d
        b_, n_, rp, ci, pt = self._csr(pat)
        self._check(fn(_i(b_), _i(n_), rp, ci, pt, ptr(A), ptr(vals), ptr(dlu), ptr(piv), ptr(dinv)))
        return dict(vals=vals, diag_lu=dlu, diag_piv=piv, diag_inv=dinv)

    def ilu_apply(self, pat, A, rhs):
        cplx = np.iscomplexobj(A)
        dt = np.complex128 if cplx else np.float64
        A = np.ascontiguousarray(A, dt)
        rhs = np.ascontiguousarray(rhs, dt)
        x = np.zeros_like(rhs)
        fn = self.lib.ref_ilu_apply_z if cplx else self.lib.ref_ilu_apply_d
        b, n, rp, ci, pt = self._csr(pat)
        self._check(fn(_i(b), _i(n), rp, ci, pt, ptr(A), ptr(rhs), ptr(x)))
        return x

    def matvec(self, pat, A, x):
        cplx = np.iscomplexobj(A) or np.iscomplexobj(x)
        dt = np.complex128 if cplx else np.float64
        A = np.ascontiguousarray(A, dt)
        x = np.ascontiguousarray(x, dt)
        y = np.zeros_like(x)
        fn = self.lib.ref_matvec_z if cplx else self.lib.ref_matvec_d
        b, n, rp, ci, _ = self._csr(pat)
        self._check(fn(_i(b), _i(n), rp, ci, ptr(A), ptr(x), ptr(y)))
        return y

    def smoothed_solve(self, pat, A, rhs, tol, max_iter, trace=False):
        cplx = np.iscomplexobj(A)
        dt = np.complex128 if cplx else np.float64
        A = np.ascontiguousarray(A, dt)
        rhs = np.ascontiguousarray(rhs, dt)
        x = np.zeros_like(rhs)
        tr = np.zeros(max_iter * len(rhs), dt) if trace else None
        it, conv = _i(), _i()
        r0, r1 = _d(), _d()
        fn = self.lib.ref_smoothed_solve_z if cplx else self.lib.ref_smoothed_solve_d
        b, n, rp, ci, pt = self._csr(pat)
        self._check(fn(_i(b), _i(n), rp, ci, pt, ptr(A), ptr(rhs), _d(tol), _i(max_iter), ptr(x), C.byref(it),
                       C.byref(r0), C.byref(r1), C.byref(conv), ptr(tr)))
        rep = (it.value, r0.value, r1.value, bool(conv.value))
        if trace:
            return x, rep, tr.reshape(max_iter, len(rhs))[: it.value]
        return x, rep

    def time_sweeps(self, pat, A, rhs, sweeps):
        cplx = np.iscomplexobj(A)
        dt = np.complex128 if cplx else np.float64
        A = np.ascontiguousarray(A, dt)
        rhs = np.ascontiguousarray(rhs, dt)
        fs = _d()
        fn = self.lib.ref_time_sweeps_z if cplx else self.lib.ref_time_sweeps_d
        b, n, rp, ci, _ = self._csr(pat)
        t = fn(_i(b), _i(n), rp, ci, ptr(A), ptr(rhs), _i(sweeps), C.byref(fs))
        return t, fs.value

    # -- full-size harmonic workers (bench.py --impl reference): the reference's own objects
    def lhs_create(self, pat, A5):
        """The shared real LHS A5 on its pattern (Bsr<real>); keep the handle alive while
        workers use it."""
        self._lhs_keep = [np.ascontiguousarray(pat["row_ptr"]), np.ascontiguousarray(pat["col_idx"]),
                          np.ascontiguousarray(A5, np.float64)]
        b, n = int(pat["b"]), len(pat["row_ptr"]) - 1
        self.lib.ref_lhs_create.restype = _p
        h = self.lib.ref_lhs_create(_i(b), _i(n), ptr(self._lhs_keep[0]), ptr(self._lhs_keep[1]), ptr(self._lhs_keep[2]))
        if not h:
            self._check(7)
        return h

    def hworker_create(self, lhs, shift_im, rhs):
        """One harmonic worker: shift_diagonal into its complex workspace + Ilu factorize.
        Returns (handle, factorization seconds)."""
        fs = _d()
        self.lib.ref_hworker_create.restype = _p
        sh = np.ascontiguousarray(shift_im, np.float64)
        r = np.ascontiguousarray(rhs, np.complex128)
        h = self.lib.ref_hworker_create(_p(lhs), ptr(sh), ptr(r), C.byref(fs))
        if not h:
            self._check(7)
        return h, fs.value

    def hworker_sweeps(self, w, sweeps):
        """smoothed_solve of `sweeps` iterations on the worker's system: (seconds, final norm)."""
        t, f = _d(), _d()
        self._check(self.lib.ref_hworker_sweeps(_p(w), _i(sweeps), C.byref(t), C.byref(f)))
        return t.value, f.value

    def hworker_destroy(self, w):
        self.lib.ref_hworker_destroy(_p(w))

    def lhs_destroy(self, h):
        self.lib.ref_lhs_destroy(_p(h))

    def build_lhs_mean(self, pat, J, implicit, sigma, eps, stage):
        A = np.zeros_like(J)
        b, n, rp, ci, _ = self._csr(pat)
        self._check(self.lib.ref_build_lhs_mean(_i(b), _i(n), rp, ci, ptr(J), _i(implicit), _d(sigma), _d(eps),
                                                _i(stage), ptr(A)))
        return A

    def cdiv(self, a, b):
        a = np.ascontiguousarray(a, np.complex128)
        b = np.ascontiguousarray(b, np.complex128)
        out = np.zeros_like(a)
        self.lib.ref_cdiv(ptr(a), ptr(b), ptr(out), _i(len(a)))
        return out

    def nozzle(self, case_text):
        return RefNozzle(self, case_text)

    def solver(self, case_text, implicit=1, sigma=-1.0, eps=0.6, tol=1e-2, max_iter=10, drop=8.0, max_outer=2000,
               mg_levels=1):
        return RefSolver(self, case_text, implicit, sigma, eps, tol, max_iter, drop, max_outer, mg_levels)


class RefNozzle:
    """The reference's quasi-1D Euler nozzle discretization, b = 3."""

    def __init__(self, ref, case_text):
        self.r = ref
        self.h = ref.lib.ref_nozzle_create(case_text.encode())
        if not self.h:
            raise CheckerError(1, ref.lib.ref_last_error().decode())
        s = np.zeros(5, np.int32)
        ref.lib.ref_nozzle_sizes(_p(self.h), ptr(s))
        self.n, self.nf, self.b, self.nnzb, self.nh = [int(x) for x in s]
        n, nf = self.n, self.nf
        self.fa = np.zeros(nf, np.int32)
        self.fb = np.zeros(nf, np.int32)
        self.fbc = np.zeros(nf, np.int32)
        self.ford = np.zeros(nf, np.int32)
        self.area = np.zeros(nf)
        self.vol = np.zeros(n)
        self.nf_ptr = np.zeros(n + 1, np.int32)
        self.nf_idx = np.zeros(2 * nf, np.int32)
        self.row_ptr = np.zeros(n + 1, np.int32)
        self.col_idx = np.zeros(self.nnzb, np.int32)
        ref.lib.ref_nozzle_mesh(_p(self.h), ptr(self.fa), ptr(self.fb), ptr(self.fbc), ptr(self.ford), ptr(self.area),
                                ptr(self.vol), ptr(self.nf_ptr), ptr(self.nf_idx), ptr(self.row_ptr),
                                ptr(self.col_idx))
        self.nf_idx = self.nf_idx[: self.nf_ptr[-1]].copy()
        cs = np.zeros(6)
        ref.lib.ref_nozzle_case(_p(self.h), ptr(cs))
        self.gamma, self.gas_constant, self.p0, self.T0, self.p_out, self.forcing_scale = cs
        self.omega = np.zeros(max(self.nh, 1))
        self.index = np.zeros(max(self.nh, 1), np.int32)
        self.forcing = np.zeros(3 * max(self.nh, 1), np.complex128)
        ref.lib.ref_nozzle_harmonics(_p(self.h), ptr(self.omega), ptr(self.index), ptr(self.forcing))
        self.omega = self.omega[: self.nh]
        self.index = self.index[: self.nh]
        self.forcing = self.forcing[: 3 * self.nh].reshape(self.nh, 3)

    def __del__(self):
        try:
            self.r.lib.ref_nozzle_destroy(_p(self.h))
        except Exception:
            pass

    def pattern(self, b=3):
        diag = np.array([self.row_ptr[i] + np.searchsorted(self.col_idx[self.row_ptr[i]:self.row_ptr[i + 1]], i)
                         for i in range(self.n)], np.int32)
        return dict(b=b, row_ptr=self.row_ptr, col_idx=self.col_idx, diag_idx=diag,
                    partition=np.zeros(self.n, np.int32))

    def initial_mean(self):
        W = np.zeros(self.n * 3)
        self.r._check(self.r.lib.ref_nozzle_initial_mean(_p(self.h), ptr(W)))
        return W

    def residual(self, W, order, mode=0, wref=None, forcing=None, need_vis=False):
        inv = np.zeros(self.n * 3)
        vis = np.zeros(self.n * 3)
        f = None if forcing is None else np.ascontiguousarray(forcing, np.float64)
        self.r._check(self.r.lib.ref_nozzle_residual(_p(self.h), ptr(np.ascontiguousarray(W)), ptr(wref), _i(order),
                                                     _i(mode), ptr(f), _i(0 if f is None else len(f)),
                                                     _i(int(need_vis)), ptr(inv), ptr(vis)))
        return inv, vis

    def jacobian(self, W):
        J = np.zeros(self.nnzb * 9)
        self.r._check(self.r.lib.ref_nozzle_jacobian(_p(self.h), ptr(np.ascontiguousarray(W)), ptr(J)))
        return J

    def diag_blocks(self, W):
        P = np.zeros(self.n * 9)
        self.r._check(self.r.lib.ref_nozzle_diag_blocks(_p(self.h), ptr(np.ascontiguousarray(W)), ptr(P)))
        return P

    def linearized_residual(self, mean, what, omega, forcing, order=2, need_vis=True):
        inv = np.zeros(self.n * 3, np.complex128)
        vis = np.zeros(self.n * 3, np.complex128)
        f = np.ascontiguousarray(forcing, np.complex128)
        self.r._check(self.r.lib.ref_nozzle_linres(_p(self.h), ptr(np.ascontiguousarray(mean)),
                                                   ptr(np.ascontiguousarray(what, np.complex128)), _d(omega), ptr(f),
                                                   _i(len(f)), _i(order), _i(int(need_vis)), ptr(inv), ptr(vis)))
        return inv, vis

    def deterministic_flux(self, mean, omegas, amps, index=None):
        nh = len(omegas)
        idx = np.arange(1, nh + 1, dtype=np.int32) if index is None else np.asarray(index, np.int32)
        df = np.zeros(self.n * 3)
        self.r._check(self.r.lib.ref_nozzle_df(_p(self.h), ptr(np.ascontiguousarray(mean)), _i(nh), ptr(idx),
                                               ptr(np.asarray(omegas, np.float64)),
                                               ptr(np.ascontiguousarray(amps, np.complex128)), ptr(df)))
        return df


class RefSolver:
    def __init__(self, ref, case_text, implicit, sigma, eps, tol, max_iter, drop, max_outer, mg_levels=1):
        self.r = ref
        self.h = ref.lib.ref_solver_create(case_text.encode(), _i(implicit), _d(sigma), _d(eps), _d(tol),
                                           _i(max_iter), _d(drop), _i(max_outer), _i(mg_levels))
        if not self.h:
            raise CheckerError(1, ref.lib.ref_last_error().decode())
        self.noz = RefNozzle(ref, case_text)

    def __del__(self):
        try:
            self.r.lib.ref_solver_destroy(_p(self.h))
        except Exception:
            pass

    def outer_iteration(self):
        e = np.zeros(4)
        rh = np.zeros(max(self.noz.nh, 1))
        self.r._check(self.r.lib.ref_solver_outer(_p(self.h), ptr(e), ptr(rh)))
        return dict(iter=int(e[0]), resid_mean=e[1], rz=e[2], has_rz=bool(e[3]), resid_h=rh[: self.noz.nh].copy())

    def state(self):
        n = self.noz.n * 3
        mean = np.zeros(n)
        amps = np.zeros(self.noz.nh * n, np.complex128)
        self.r.lib.ref_solver_state(_p(self.h), ptr(mean), ptr(amps))
        return mean, amps.reshape(self.noz.nh, n)

    def df(self):
        d = np.zeros(self.noz.n * 3)
        self.r.lib.ref_solver_df(_p(self.h), ptr(d))
        return d

    def run(self, max_hist=100000, max_rep=1000000):
        nh_, nr = _i(), _i()
        hist = np.zeros(3 * max_hist)
        reps = np.zeros(4 * max_rep)
        peak = _d()
        reason = self.r.lib.ref_solver_run(_p(self.h), C.byref(nh_), ptr(hist), _i(max_hist), C.byref(nr), ptr(reps),
                                           _i(max_rep), C.byref(peak))
        if reason < 0:
            raise CheckerError(99, self.r.lib.ref_last_error().decode())
        return dict(reason=reason, history=hist[: 3 * nh_.value].reshape(-1, 3),
                    reports=reps[: 4 * nr.value].reshape(-1, 4), peak_lhs_bytes=peak.value)
