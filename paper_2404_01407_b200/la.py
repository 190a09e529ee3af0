"""Python mirror of the reference's block-sparse LA operators (sparse.hpp), backed by
the device kernels through the C ABI.  Argument meaning and error behaviour follow
the reference: ``FnlhError`` carries ConfigError / FactorizationError(node) /
DivergenceError(stage) exactly where the reference throws them."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import LinearReport, as_pairs, check, f64, lib, ptr

_i, _d = C.c_int, C.c_double


class Pattern:
    """BlockSparsityPattern (sparse.hpp:106-121) resident on the device."""

    def __init__(self, b, row_ptr, col_idx, partition=None):
        self.b = int(b)
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int32)
        self.col_idx = np.ascontiguousarray(col_idx, np.int32)
        self.partition = None if partition is None else np.ascontiguousarray(partition, np.int32)
        self.rows = len(self.row_ptr) - 1
        self.nnzb = len(self.col_idx)
        h = C.c_void_p()
        check(lib().fnlh_pattern_create(_i(self.b), _i(self.rows), ptr(self.row_ptr), ptr(self.col_idx),
                                        ptr(self.partition), C.byref(h)))
        self.h = h

    @classmethod
    def from_dict(cls, pat):
        return cls(pat["b"], pat["row_ptr"], pat["col_idx"], pat.get("partition"))

    def levels(self):
        f, b = _i(), _i()
        lib().fnlh_pattern_levels(self.h, C.byref(f), C.byref(b))
        return f.value, b.value

    def __del__(self):
        try:
            lib().fnlh_pattern_destroy(self.h)
        except Exception:
            pass


def _system(A, shift_im):
    """-> (is_complex, A buffer, A_complex flag, shift buffer)"""
    if np.iscomplexobj(A):
        return 1, as_pairs(A), 1, None
    if shift_im is not None:
        return 1, f64(A), 0, f64(shift_im)
    return 0, f64(A), 0, None


def ilu_factorize(pat: Pattern, A, shift_im=None):
    """Ilu<S>::factorize (sparse.cpp:187-257); A complex, or real A5 (+ per-node i*shift)."""
    cplx, Ab, Ac, sh = _system(A, shift_im)
    dt = np.complex128 if cplx else np.float64
    b, n = pat.b, pat.rows
    vals = np.zeros(pat.nnzb * b * b, dt)
    dlu = np.zeros(n * b * b, dt)
    piv = np.zeros(n * b, np.int32)
    dinv = np.zeros(n * b * b, dt)
    v = (lambda a: a.view(np.float64)) if cplx else (lambda a: a)
    check(lib().fnlh_ilu_factorize(pat.h, _i(cplx), ptr(Ab), _i(Ac), ptr(sh), ptr(v(vals)), ptr(v(dlu)), ptr(piv),
                                   ptr(v(dinv))))
    return dict(vals=vals, diag_lu=dlu, diag_piv=piv, diag_inv=dinv)


def ilu_apply(pat: Pattern, A, rhs, shift_im=None):
    cplx, Ab, Ac, sh = _system(A, shift_im)
    if cplx:
        r = as_pairs(rhs)
        x = np.zeros(pat.rows * pat.b, np.complex128)
        check(lib().fnlh_ilu_apply(pat.h, _i(1), ptr(Ab), _i(Ac), ptr(sh), ptr(r), ptr(x.view(np.float64))))
    else:
        r = f64(rhs)
        x = np.zeros(pat.rows * pat.b)
        check(lib().fnlh_ilu_apply(pat.h, _i(0), ptr(Ab), _i(0), None, ptr(r), ptr(x)))
    return x


def matvec(pat: Pattern, A, x, shift_im=None):
    cplx, Ab, Ac, sh = _system(A, shift_im)
    if cplx or np.iscomplexobj(x):
        if not cplx:
            cplx, Ab, Ac = 1, f64(A), 0
        xv = as_pairs(x)
        y = np.zeros(pat.rows * pat.b, np.complex128)
        check(lib().fnlh_matvec(pat.h, _i(1), ptr(Ab), _i(Ac), ptr(sh), ptr(xv), ptr(y.view(np.float64))))
    else:
        y = np.zeros(pat.rows * pat.b)
        check(lib().fnlh_matvec(pat.h, _i(0), ptr(Ab), _i(0), None, ptr(f64(x)), ptr(y)))
    return y


def smoothed_solve(pat: Pattern, A, rhs, tol_rel, max_iter, shift_im=None):
    """factorize + smoothed_solve (sparse.hpp:295-331) -> (x, (iterations, r0, r1, converged))"""
    cplx, Ab, Ac, sh = _system(A, shift_im)
    rep = LinearReport()
    if cplx:
        x = np.zeros(pat.rows * pat.b, np.complex128)
        check(lib().fnlh_smoothed_solve(pat.h, _i(1), ptr(Ab), _i(Ac), ptr(sh), ptr(as_pairs(rhs)), _d(tol_rel),
                                        _i(max_iter), ptr(x.view(np.float64)), C.byref(rep)))
    else:
        x = np.zeros(pat.rows * pat.b)
        check(lib().fnlh_smoothed_solve(pat.h, _i(0), ptr(Ab), _i(0), None, ptr(f64(rhs)), _d(tol_rel), _i(max_iter),
                                        ptr(x), C.byref(rep)))
    return x, rep.as_tuple()


def set_graphs(enable: bool):
    """CUDA-graph replay of the outer iteration's synchronization-free launch sequences
    (include/fnlh_b200.h fnlh_set_graphs); off = launch by launch, same results."""
    lib().fnlh_set_graphs(_i(1 if enable else 0))


def set_red_black(enable: bool):
    """Enable / disable the 2-colour fused sweep (rb.cuh) in favour of the level-scheduled kernels."""
    lib().fnlh_set_red_black(_i(1 if enable else 0))


RB_EXACT, RB_EXACT_SPLIT, RB_ONEPASS, RB_EDGE, RB_LANEWARP, RB_STAGED, RB_ASTAGED = 0, 1, 2, 3, 4, 5, 6


def set_rb_sweep(mode: int):
    """2-colour sweep variant (include/fnlh_b200.h fnlh_set_rb_sweep): RB_EXACT (default,
    bitwise reference iterates, 2 kernels/sweep), RB_EXACT_SPLIT (same, 3 kernels/sweep),
    RB_ONEPASS (one pass over A, iterates equal to rounding), RB_EDGE (bitwise, the colour-1
    kernel edge-parallel: one thread per (row, lower block)), RB_LANEWARP / RB_STAGED /
    RB_ASTAGED (bitwise; batches of P > 1 systems: lane-warp CTAs, with A in shared memory and a
    cp.async ring for inv(U_kk), or A in shared memory only) -- measured variants, DESIGN 4.1."""
    check(lib().fnlh_set_rb_sweep(_i(mode)))


def red_black_n0(pat: Pattern) -> int:
    """Size of colour 0 if the pattern is a colour-major 2-colour ordering with one partition, else -1."""
    n0 = _i()
    check(lib().fnlh_pattern_is_red_black(pat.h, C.byref(n0)))
    return n0.value


def rb_factorize(pat: Pattern, A, shift_im=None):
    """Compact 2-colour ILU(0) factors: pivot LU + piv for all rows, inv(U_kk) for colour 0."""
    n0 = red_black_n0(pat)
    cplx = shift_im is not None
    dt = np.complex128 if cplx else np.float64
    b, n = pat.b, pat.rows
    dlu = np.zeros(n * b * b, dt)
    piv = np.zeros(n * b, np.int32)
    inv0 = np.zeros(max(n0, 1) * b * b, dt)
    v = (lambda a: a.view(np.float64)) if cplx else (lambda a: a)
    check(lib().fnlh_rb_factorize(pat.h, _i(1 if cplx else 0), ptr(f64(A)), ptr(None if shift_im is None else f64(shift_im)),
                                  ptr(v(dlu)), ptr(piv), ptr(v(inv0))))
    return dict(diag_lu=dlu, diag_piv=piv, inv0=inv0[: n0 * b * b], n0=n0)


class Lhs:
    """The shared real LHS (Bsr<real> A5, sparse.hpp:136-157) resident on the device
    (include/fnlh_b200.h fnlh_lhs): uploaded once, read by any number of Ilu workspaces."""

    def __init__(self, pat: Pattern, A=None):
        self.pat = pat
        h = C.c_void_p()
        check(lib().fnlh_lhs_create(pat.h, C.byref(h)))
        self.h = h
        if A is not None:
            self.upload(A)

    def upload(self, A):
        check(lib().fnlh_lhs_upload(self.h, ptr(f64(A))))

    def bytes(self):
        v = C.c_longlong()
        check(lib().fnlh_lhs_bytes(self.h, C.byref(v)))
        return v.value

    def __del__(self):
        try:
            lib().fnlh_lhs_destroy(self.h)
        except Exception:
            pass


class Ilu:
    """One worker's Ilu<S> workspace on a device Lhs (fnlh_prec): factorize() for the real
    operator (Ilu<real>, the mean flow), factorize(shift_im) for the harmonic operator
    A5 + i diag(shift_im) (build_lhs_harmonic + Ilu<cplx>::factorize, driver.cpp:213-216);
    solve() is smoothed_solve on the resident factors (rk.cpp:82-85)."""

    def __init__(self, A: Lhs, is_complex: bool):
        self.A = A
        self.cplx = bool(is_complex)
        h = C.c_void_p()
        check(lib().fnlh_prec_create(A.h, _i(1 if is_complex else 0), C.byref(h)))
        self.h = h

    def factorize(self, shift_im=None):
        sh = None if shift_im is None else f64(shift_im)
        check(lib().fnlh_prec_factorize(self.h, ptr(sh)))

    def solve(self, rhs, tol_rel, max_iter):
        """-> (x, (iterations, initial norm, final norm, converged))"""
        if self.cplx:
            r = as_pairs(rhs)
            x = np.zeros(len(r) // 2, np.complex128)
        else:
            r = f64(rhs)
            x = np.zeros(len(r))
        rep = LinearReport()
        check(lib().fnlh_richardson(self.h, ptr(r), _d(tol_rel), _i(max_iter), ptr(x.view(np.float64)),
                                    C.byref(rep)))
        return x, rep.as_tuple()

    def bytes(self):
        v = C.c_longlong()
        check(lib().fnlh_prec_bytes(self.h, C.byref(v)))
        return v.value

    def __del__(self):
        try:
            lib().fnlh_prec_destroy(self.h)
        except Exception:
            pass
