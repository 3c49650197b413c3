"""ORACLE (test infrastructure only) — ctypes wrapper of oracle/c/oracle.c."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "c", "oracle.c")
LIB = os.path.join(_HERE, "c", "liboracle.so")
FORM_ID = {"mod": 0, "sym": 1, "grad": 2}
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", LIB, SRC, "-lm"])
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        L.ora_apply_slab.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, P, P, P, P, P,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_uint]
        L.ora_diag.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, P, P, P, P, P]
        L.ora_apply_rows.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, P, P, P, P, P,
                                     ctypes.c_int64, P]
        L.ora_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _coef(cls, class_mu, mu_a, imu_c):
    """Per-element (mu_A, 1/mu_C) arrays: from the classes on the finest level, or
    given directly (coarse levels, reading R15)."""
    if mu_a is None:
        mu_a = np.asarray(class_mu, dtype=np.float64)[np.asarray(cls)]
        imu_c = 1.0 / mu_a
    return (np.ascontiguousarray(mu_a, dtype=np.float64).reshape(-1),
            np.ascontiguousarray(imu_c, dtype=np.float64).reshape(-1))


def apply_slab(n, form, delta, faces, cls, class_mu, x, kv0=0, kv1=None, y=None, blocks=15,
               mu_a=None, imu_c=None):
    """y = K x for the rows of vertex planes [kv0, kv1); x, y field-major (4, V)."""
    kv1 = n + 1 if kv1 is None else kv1
    V = (n + 1) ** 3
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(4 * V)
    y = np.zeros(4 * V) if y is None else y
    f = np.ascontiguousarray(faces, dtype=np.int32)
    c, m = _coef(cls, class_mu, mu_a, imu_c)
    lib().ora_apply_slab(n, FORM_ID[form], float(delta), _p(f), _p(c), _p(m), _p(x), _p(y), kv0, kv1,
                         blocks)
    return y


def diagonals(n, form, delta, faces, cls, class_mu, mu_a=None, imu_c=None):
    """(diag A (3V,), diag C (V,)) by the element loop."""
    V = (n + 1) ** 3
    dA = np.zeros(3 * V)
    dC = np.zeros(V)
    f = np.ascontiguousarray(faces, dtype=np.int32)
    c, m = _coef(cls, class_mu, mu_a, imu_c)
    lib().ora_diag(n, FORM_ID[form], float(delta), _p(f), _p(c), _p(m), _p(dA), _p(dC))
    return dA, dC


def apply_rows(n, form, delta, faces, cls, class_mu, x, verts, mu_a=None, imu_c=None):
    """(len(verts), 4) rows of K x at the listed vertex ids."""
    V = (n + 1) ** 3
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(4 * V)
    verts = np.ascontiguousarray(verts, dtype=np.int64)
    out = np.zeros((len(verts), 4))
    f = np.ascontiguousarray(faces, dtype=np.int32)
    c, m = _coef(cls, class_mu, mu_a, imu_c)
    lib().ora_apply_rows(n, FORM_ID[form], float(delta), _p(f), _p(c), _p(m), _p(x), _p(verts),
                         len(verts), _p(out))
    return out


def num_threads() -> int:
    return lib().ora_num_threads()
