"""Python mirror of the reference's operator / solver interface (disc.hpp,
residual_ops.hpp, driver.hpp) over the device C ABI.  Names, argument meaning and
error behaviour follow the reference; arrays use its layouts (node-major AoS)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import FnlhError, LinearReport, as_pairs, check, f64, lib, ptr

_i, _d, _p = C.c_int, C.c_double, C.c_void_p


class MeshDesc(C.Structure):
    _fields_ = [("n", _i), ("nf", _i), ("b", _i), ("fa", _p), ("fb", _p), ("fbc", _p), ("ford", _p), ("fn", _p),
                ("farea", _p), ("fnh", _p), ("fvis", _p), ("vol", _p), ("closure", _p), ("mu", _p), ("nf_ptr", _p),
                ("nf_idx", _p), ("bflag", _p), ("gamma", _d), ("gas_constant", _d), ("p0", _d), ("T0", _d),
                ("p_out", _d), ("nt_in", _d), ("forcing_scale", _d)]


class Scheme(C.Structure):
    _fields_ = [("implicit", _i), ("sigma_cfl", _d), ("eps_relax", _d), ("linear_tol", _d), ("linear_max_iter", _i),
                ("target_drop_orders", _d), ("max_outer_iters", _i), ("workers", _i)]


class Entry(C.Structure):
    _fields_ = [("iter", _i), ("resid_mean", _d), ("rz", _d), ("has_rz", _i), ("seconds", _d)]


def _desc(m, keep):
    arrs = [m.fa, m.fb, m.fbc, m.ford, m.fn, m.farea, m.fnh, m.fvis, m.vol, m.closure, m.mu, m.nf_ptr, m.nf_idx,
            m.bflag]
    keep.extend(arrs)
    return MeshDesc(m.n, m.nf, m.b, *[ptr(a) for a in arrs], m.gamma, m.gas_constant, m.p0, m.T0, m.p_out, m.nt_in,
                    m.forcing_scale)


def scheme_struct(s: dict) -> Scheme:
    return Scheme(int(s.get("implicit", 1)), float(s.get("sigma_cfl", -1.0)), float(s.get("eps_relax", 0.6)),
                  float(s.get("linear_tol", 1e-2)), int(s.get("linear_max_iter", 10)),
                  float(s.get("target_drop_orders", 8.0)), int(s.get("max_outer_iters", 2000)),
                  int(s.get("workers", 1)))


class Discretization:
    """Device-resident 3D edge-based discretization (disc.hpp:42-106 operator contract)."""

    def __init__(self, mesh, pattern=None):
        self.m = mesh
        self._keep = []
        pat = pattern or mesh.pattern()
        self._keep += [pat["row_ptr"], pat["col_idx"], pat["partition"]]
        self.desc = _desc(mesh, self._keep)
        h = _p()
        check(lib().fnlh_disc_create(C.byref(self.desc), ptr(pat["row_ptr"]), ptr(pat["col_idx"]),
                                     ptr(pat["partition"]), C.byref(h)))
        self.h = h
        self.pattern = pat

    def __del__(self):
        try:
            lib().fnlh_disc_destroy(self.h)
        except Exception:
            pass

    def residual(self, W, order, mode=0, wref=None, forcing=None, need_vis=False):
        n = self.m.n * self.m.b
        inv, vis = np.zeros(n), np.zeros(n)
        f = None if forcing is None else f64(forcing)
        check(lib().fnlh_disc_residual(self.h, ptr(f64(W)), ptr(None if wref is None else f64(wref)), _i(order),
                                       _i(mode), ptr(f), _i(0 if f is None else len(f)), _i(int(need_vis)), ptr(inv),
                                       ptr(vis)))
        return inv, vis

    def fd_jacobian(self, W, want_J=True, want_P=False):
        b = self.m.b
        J = np.zeros(len(self.pattern["col_idx"]) * b * b) if want_J else None
        P = np.zeros(self.m.n * b * b) if want_P else None
        check(lib().fnlh_disc_fd_jacobian(self.h, ptr(f64(W)), ptr(J), ptr(P)))
        return J, P

    def linearized_residual(self, mean, what, omega, forcing, order=2, need_vis=True):
        n = self.m.n * self.m.b
        inv = np.zeros(n, np.complex128)
        vis = np.zeros(n, np.complex128)
        f = as_pairs(forcing)
        check(lib().fnlh_disc_linearized_residual(self.h, ptr(f64(mean)), ptr(as_pairs(what)), _d(omega), ptr(f),
                                                  _i(len(f) // 2), _i(order), _i(int(need_vis)),
                                                  ptr(inv.view(np.float64)), ptr(vis.view(np.float64))))
        return inv, vis

    def deterministic_flux(self, mean, omegas, amps):
        df = np.zeros(self.m.n * self.m.b)
        om = f64(omegas)
        check(lib().fnlh_disc_deterministic_flux(self.h, ptr(f64(mean)), _i(len(om)), ptr(om), ptr(as_pairs(amps)),
                                                 ptr(df)))
        return df


class FnlhSolver:
    """FnlhSolver (driver.hpp:83-126) on the device: outer_iteration / run_to_convergence."""

    def __init__(self, mesh, scheme: dict, omegas, forcing, mean0, index=None, pattern=None):
        self.m = mesh
        self.nh = len(omegas)
        self._keep = []
        pat = pattern or mesh.pattern()
        self._keep += [pat["row_ptr"], pat["col_idx"], pat["partition"]]
        self.desc = _desc(mesh, self._keep)
        self.scheme = scheme_struct(scheme)
        idx = np.arange(1, self.nh + 1, dtype=np.int32) if index is None else np.asarray(index, np.int32)
        om = f64(omegas)
        fz = np.asarray(forcing, np.complex128).reshape(self.nh, -1) if self.nh else np.zeros((0, 0), np.complex128)
        nforcing = fz.shape[1] if self.nh else 0
        forc = as_pairs(fz.reshape(-1)) if fz.size else np.zeros(2)
        self._keep += [idx, om, forc]
        h = _p()
        check(lib().fnlh_solver_create(C.byref(self.desc), ptr(pat["row_ptr"]), ptr(pat["col_idx"]),
                                       ptr(pat["partition"]), C.byref(self.scheme), _i(self.nh), ptr(idx), ptr(om),
                                       ptr(forc), _i(nforcing), ptr(f64(mean0)), C.byref(h)))
        self.h = h
        self.omegas = np.array(om)
        self.hierarchy = None
        levels = int(scheme.get("mg_levels", 1))
        if levels > 1:  # SchemeConfig::mg_levels (driver.hpp:24): 2x2x2 agglomeration, mesh.hierarchy
            from .mesh import hierarchy
            self.hierarchy = hierarchy(mesh, levels, fz if self.nh else None)
            for lv in range(1, levels):
                self.add_level(self.hierarchy[lv][0], self.hierarchy[lv - 1][1], self.hierarchy[lv][2])

    def add_level(self, mesh, parent, forcing=None):
        """Append a coarse multigrid level (explicit scheme): its mesh, parent[i] = its node
        agglomerating node i of the current coarsest level, its boundary forcing [nh, nf]."""
        pat = mesh.pattern()
        par = np.ascontiguousarray(parent, np.int32)
        fz = np.asarray(forcing, np.complex128).reshape(self.nh, -1) if (self.nh and forcing is not None) else \
            np.zeros((self.nh, 0), np.complex128)
        forc = as_pairs(fz.reshape(-1)) if fz.size else np.zeros(2)
        keep = [pat["row_ptr"], pat["col_idx"], par, forc]
        desc = _desc(mesh, keep)
        self._keep += keep + [desc]
        check(lib().fnlh_solver_add_level(self.h, C.byref(desc), ptr(pat["row_ptr"]), ptr(pat["col_idx"]), ptr(par),
                                          ptr(forc), _i(fz.shape[1] if self.nh else 0)))

    def levels(self):
        return lib().fnlh_solver_levels(self.h)

    def __del__(self):
        try:
            lib().fnlh_solver_destroy(self.h)
        except Exception:
            pass

    def outer_iteration(self):
        e = Entry()
        rh = np.zeros(max(self.nh, 1))
        check(lib().fnlh_solver_outer_iteration(self.h, C.byref(e), ptr(rh)))
        return dict(iter=e.iter, resid_mean=e.resid_mean, rz=e.rz, has_rz=bool(e.has_rz), resid_h=rh[: self.nh].copy(),
                    seconds=e.seconds)

    def outer_iteration_host(self, mean_in, amps_in, mean_out=None, amps_out=None):
        """outer_iteration on host buffers (upload, step, download overlapped); the output
        arrays default to the inputs (in place).  Pinned arrays make the copies async."""
        mean_out = mean_in if mean_out is None else mean_out
        amps_out = amps_in if amps_out is None else amps_out
        for a in (mean_in, amps_in, mean_out, amps_out):
            assert a.flags.c_contiguous
        assert mean_in.dtype == np.float64 and amps_in.dtype == np.complex128
        e = Entry()
        rh = np.zeros(max(self.nh, 1))
        check(lib().fnlh_solver_outer_iteration_host(self.h, ptr(mean_in), ptr(amps_in.reshape(-1).view(np.float64)),
                                                     ptr(mean_out), ptr(amps_out.reshape(-1).view(np.float64)),
                                                     C.byref(e), ptr(rh)))
        return dict(iter=e.iter, resid_mean=e.resid_mean, rz=e.rz, has_rz=bool(e.has_rz), resid_h=rh[: self.nh].copy(),
                    seconds=e.seconds)

    # the two halves of outer_iteration (harmonic sharding across GPUs, shard.py)
    def phase_harmonics(self, owned=None):
        hn = np.zeros(max(self.nh, 1))
        own = None if owned is None else np.ascontiguousarray(owned, np.int32)
        check(lib().fnlh_solver_phase_harmonics(self.h, ptr(own), ptr(hn)))
        return hn[: self.nh].copy()

    # deterministic_flux split over quadrature points (shard.py; include/fnlh_b200.h)
    def df_points(self):
        nq = _i()
        check(lib().fnlh_solver_df_points(self.h, C.byref(nq)))
        return nq.value

    def df_terms(self, k0, k1, terms_ptr):
        check(lib().fnlh_solver_df_terms(self.h, _i(k0), _i(k1), C.c_void_p(terms_ptr)))

    def df_accumulate(self, terms_ptr, count, acc_ptr, first):
        check(lib().fnlh_solver_df_accumulate(self.h, C.c_void_p(terms_ptr), _i(count), C.c_void_p(acc_ptr),
                                              _i(1 if first else 0)))

    def set_external_df(self, acc_ptr):
        check(lib().fnlh_solver_set_external_df(self.h, C.c_void_p(acc_ptr)))

    def failed_harmonic(self):
        """Harmonic whose error the last phase_harmonics raised (-1: none / before the harmonics)."""
        h = _i()
        check(lib().fnlh_solver_failed_harmonic(self.h, C.byref(h)))
        return h.value

    def harmonic_reports(self, h):
        arr = (LinearReport * 256)()
        n = _i()
        check(lib().fnlh_solver_harmonic_reports(self.h, _i(h), arr, _i(256), C.byref(n)))
        return [r.as_tuple() for r in arr[: n.value]]

    def phase_mean(self, h_norm, h_reports):
        reps = [r for hr in h_reports for r in hr]
        arr = (LinearReport * max(len(reps), 1))(*[LinearReport(r[0], r[1], r[2], int(r[3])) for r in reps])
        nrep = np.array([len(hr) for hr in h_reports] + [0], np.int32)
        e = Entry()
        rh = np.zeros(max(self.nh, 1))
        check(lib().fnlh_solver_phase_mean(self.h, ptr(f64(h_norm)), ptr(nrep), arr, C.byref(e), ptr(rh)))
        return dict(iter=e.iter, resid_mean=e.resid_mean, rz=e.rz, has_rz=bool(e.has_rz), resid_h=rh[: self.nh].copy(),
                    seconds=e.seconds)

    def copy_amps(self, h, dev_ptr, to_dev):
        """Device-to-device copy of harmonic h's field to (to_dev) / from caller memory."""
        check(lib().fnlh_solver_copy_amps(self.h, _i(h), C.c_void_p(dev_ptr), _i(1 if to_dev else 0)))

    def run_to_convergence(self, max_entries=100000):
        reason, n = _i(), _i()
        arr = (Entry * max_entries)()
        check(lib().fnlh_solver_run(self.h, C.byref(reason), C.byref(n), arr, _i(max_entries)))
        hist = [dict(iter=e.iter, resid_mean=e.resid_mean, rz=e.rz, seconds=e.seconds) for e in arr[: min(n.value, max_entries)]]
        return ["target-drop", "iteration-cap", "divergence"][reason.value], hist

    def state(self, out=None):
        """(mean, amps); `out` = preallocated (mean [N b] f64, amps [N_h, N b] c128) host
        arrays (e.g. pinned) to download into."""
        n = self.m.n * self.m.b
        if out is not None:
            mean, amps = out
            assert mean.flags.c_contiguous and amps.flags.c_contiguous and amps.dtype == np.complex128
            check(lib().fnlh_solver_get_state(self.h, ptr(mean), ptr(amps.reshape(-1).view(np.float64))))
            return mean, amps
        mean = np.zeros(n)
        amps = np.zeros(max(self.nh, 1) * n, np.complex128)
        check(lib().fnlh_solver_get_state(self.h, ptr(mean), ptr(amps.view(np.float64))))
        return mean, amps[: self.nh * n].reshape(self.nh, n)

    def set_state(self, mean, amps):
        check(lib().fnlh_solver_set_state(self.h, ptr(f64(mean)), ptr(as_pairs(amps))))

    def df(self):
        d = np.zeros(self.m.n * self.m.b)
        check(lib().fnlh_solver_get_df(self.h, ptr(d)))
        return d

    def reports(self):
        k = lib().fnlh_solver_num_reports(self.h)
        arr = (LinearReport * max(k, 1))()
        lib().fnlh_solver_get_reports(self.h, arr)
        return [r.as_tuple() for r in arr[:k]]

    def lhs_bytes(self):
        lib().fnlh_solver_lhs_bytes.restype = _d
        return int(lib().fnlh_solver_lhs_bytes(self.h))

    def lanes(self):
        """Harmonics in flight (min(workers, N_h, 8) on the 2-colour path, else 1)."""
        return lib().fnlh_solver_lanes(self.h)

    def time_sweeps_batch(self, P, sweeps):
        """Device ms of `sweeps` batched sweeps of harmonics [0, P)."""
        ms = _d()
        check(lib().fnlh_solver_time_sweeps_batch(self.h, _i(P), _i(sweeps), C.byref(ms)))
        return ms.value

    def time_sweeps(self, h, sweeps):
        ms = _d()
        check(lib().fnlh_solver_time_sweeps(self.h, _i(h), _i(sweeps), C.byref(ms)))
        return ms.value

    def info(self):
        out = np.zeros(4)
        check(lib().fnlh_solver_info(self.h, ptr(out)))
        return dict(red_black=bool(out[0]), n0=int(out[1]), sell_vals=int(out[2]), nnzb=int(out[3]))

    def counters(self):
        out = np.zeros(7)
        lib().fnlh_solver_counters(self.h, ptr(out))
        return dict(sweeps=int(out[0]), row_updates=int(out[1]), last_ms=float(out[2]),
                    phase_ms=dict(lhs=float(out[3]), harmonics=float(out[4]), df=float(out[5]), mean=float(out[6])))


__all__ = ["Discretization", "FnlhSolver", "FnlhError"]
