"""ctypes wrapper of oracle/frontier.c — test infrastructure only.

The row-frontier DP of oracle/frontier.py in plain C (sorted state arrays, 128-bit values),
for the matrices the Python version is too slow for (configs[4]'s n = 96 workloads).  Not a
method of the paper: an independent exact algorithm that pins per(A) (Eq. (1)).
Pinned in tests/test_oracle.py against per(C100) = Table T12's Total, brute
force and the Python DP.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "frontier.c")
_LIB = os.path.join(_HERE, "libfrontier.so")
_lib = None


def build_frontier_c(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_frontier_c()
        lib = ctypes.CDLL(_LIB)
        lib.frontier_per.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p]
        lib.frontier_per.restype = ctypes.c_int
        _lib = lib
    return _lib


def per_frontier_c(a, row_order: Sequence[int] = None, return_states: bool = False):
    """per(A) by the C frontier DP, rows taken in `row_order` (default natural)."""
    lib = _load()
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
    n = a.shape[0]
    order = np.ascontiguousarray(np.arange(n) if row_order is None else np.asarray(row_order), dtype=np.int32)
    if sorted(order.tolist()) != list(range(n)):
        raise ValueError("row_order must be a permutation")
    out = np.zeros(2, dtype=np.uint64)
    ms = np.zeros(1, dtype=np.uint64)
    rc = lib.frontier_per(n, a.ctypes.data, order.ctypes.data, out.ctypes.data, ms.ctypes.data)
    if rc != 0:
        raise ValueError(f"frontier_per failed ({rc})")
    v = int(out[0]) | (int(out[1]) << 64)
    if v >> 127:
        v -= 1 << 128
    return (v, int(ms[0])) if return_states else v


def narrow_order(a) -> list:
    """A row order that keeps the set of open columns small: greedily take the row that
    leaves the fewest open columns (ties: most columns shared with the processed rows, then
    lowest index), from every start row; keep the order with the smallest peak open count.
    Any order gives the same per(A); this one only decides how long the DP takes."""
    a = np.asarray(a)
    n = a.shape[0]
    cols = [frozenset(np.nonzero(a[i])[0].tolist()) for i in range(n)]
    rows_of = [frozenset(np.nonzero(a[:, j])[0].tolist()) for j in range(n)]
    best = None
    for start in range(n):
        done, touched, order = set(), set(), []
        cur, peak = start, 0
        while True:
            order.append(cur)
            done.add(cur)
            touched |= cols[cur]
            peak = max(peak, sum(1 for j in touched if not rows_of[j] <= done))
            if len(order) == n:
                break

            def score(i):
                d = done | {i}
                t = touched | cols[i]
                return (sum(1 for j in t if not rows_of[j] <= d), -len(cols[i] & touched), i)
            cur = min((i for i in range(n) if i not in done), key=score)
        if best is None or peak < best[0]:
            best = (peak, order)
    return best[1]
