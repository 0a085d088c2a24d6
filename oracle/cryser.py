"""ctypes wrapper of oracle/ryser_nw.c — test infrastructure only.

build_oracle_c() compiles the C oracle with plain `gcc -O2` (called by
__graft_entry__.build(); compiling the checker is not using it).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ryser_nw.c")
_LIB = os.path.join(_HERE, "libryser_nw.so")
_lib = None


def build_oracle_c(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_oracle_c()
        lib = ctypes.CDLL(_LIB)
        lib.ryser_nw_range.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64,
                                       ctypes.c_uint64, ctypes.c_void_p]
        lib.ryser_nw_range.restype = ctypes.c_int
        lib.ryser_nw_limbs.restype = ctypes.c_int
        _lib = lib
    return _lib


def ryser_nw_partial(a, t0: int, t1: int) -> int:
    """Signed exact sum of the R-NW terms t in [t0, t1) (unscaled)."""
    lib = _load()
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
    n = a.shape[0]
    L = lib.ryser_nw_limbs()
    acc = np.zeros(L, dtype=np.uint64)
    rc = lib.ryser_nw_range(n, a.ctypes.data, t0, t1, acc.ctypes.data)
    if rc != 0:
        raise ValueError("ryser_nw_range: unsupported input")
    v = 0
    for k in range(L - 1, -1, -1):
        v = (v << 64) | int(acc[k])
    if v >> (64 * L - 1):
        v -= 1 << (64 * L)
    return v


def per_ryser_nw_c(a) -> int:
    """per(A) by the C R-NW oracle over the full Gray range."""
    a = np.asarray(a, dtype=np.int64)
    n = a.shape[0]
    if n == 0:
        return 1
    s = ryser_nw_partial(a, 0, 1 << (n - 1))
    num = (-1) ** (n - 1) * s
    den = 1 << (n - 1)
    if num % den:
        raise ArithmeticError("R-NW sum not divisible by 2^(n-1)")
    return num // den
