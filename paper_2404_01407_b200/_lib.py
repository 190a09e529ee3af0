"""ctypes loader for libfnlh_b200.so (the C ABI in include/fnlh_b200.h).

There is no CPU fallback: if the extension is missing or no CUDA device is present,
every product call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FNLH_B200_LIB", os.path.join(HERE, "libfnlh_b200.so"))

_i, _d, _p = C.c_int, C.c_double, C.c_void_p

STATUS = {1: "ConfigError", 2: "StateError", 3: "ShapeError", 4: "UnsupportedCaseError",
          5: "FactorizationError", 6: "DivergenceError", 7: "CudaError", 8: "NonConvergenceError"}


class FnlhError(RuntimeError):
    """Reference exception taxonomy (core.hpp:22-56) carried through the C ABI."""

    def __init__(self, code, msg, node=-1, stage=-1):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code, self.kind, self.node, self.stage = code, STATUS.get(code, str(code)), node, stage


class LinearReport(C.Structure):
    _fields_ = [("iterations", _i), ("initial_residual", _d), ("final_residual", _d), ("converged", _i)]

    def as_tuple(self):
        return (self.iterations, self.initial_residual, self.final_residual, bool(self.converged))


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.fnlh_last_error.restype = C.c_char_p
        L.fnlh_launch_count.restype = C.c_longlong
        L.fnlh_pow_mode_info.restype = C.c_char_p
        L.fnlh_pow.restype = C.c_double
        L.fnlh_pow.argtypes = [C.c_double, C.c_double]
        _LIB = L
    return _LIB


def check(st):
    if st:
        L = lib()
        raise FnlhError(st, L.fnlh_last_error().decode(), L.fnlh_last_error_node(), L.fnlh_last_error_stage())


def pow_mode():
    """The device's boundary-state pow: "glibc" (the reference's libm restated bit for bit,
    csrc/libm_pow.cuh) or "cr" (correctly rounded; FNLH_POW=cr or the libm check failed)."""
    return "glibc" if lib().fnlh_pow_mode() == 0 else "cr"


def require_gpu():
    n = lib().fnlh_device_count()
    if n < 1:
        raise RuntimeError("no CUDA device visible: the FNLH B200 path has no CPU fallback")
    return n


def ptr(a):
    return None if a is None else a.ctypes.data_as(_p)


def f64(a):
    return np.ascontiguousarray(a, np.float64)


def as_pairs(a):
    """complex128 array -> interleaved float64 view (std::complex<double> layout)."""
    a = np.ascontiguousarray(a, np.complex128)
    return a.view(np.float64)
