"""Kendall rank correlation, Eqs. (7)-(10) of the paper — test
infrastructure only.

Written out as the definition: every pair i < j is scored a_ij = sign(x_j - x_i),
b_ij = sign(y_j - y_i) (0 for a tie), S = sum_{i<j} a_ij b_ij (Eq. 7's numerator); T and U
count the tied pairs of each ranking, T = 1/2 sum_t t(t-1) over the groups of ties (Eqs. 8, 9);
tau = S / (sqrt(n(n-1)/2 - T) sqrt(n(n-1)/2 - U)) (Eq. 10; = Eq. 7 without ties).  O(m^2).
"""
from __future__ import annotations

import math
from collections import Counter
from typing import Sequence, Tuple


def _sign(v: float) -> int:
    return int(v > 0) - int(v < 0)


def kendall_s(x: Sequence[float], y: Sequence[float]) -> int:
    n = len(x)
    return sum(_sign(x[j] - x[i]) * _sign(y[j] - y[i]) for i in range(n) for j in range(i + 1, n))


def tie_pairs(v: Sequence[float]) -> int:
    """1/2 sum_t t(t-1) over the groups of equal values (Eqs. (8), (9))."""
    return sum(t * (t - 1) // 2 for t in Counter(v).values())


def kendall_tau_b(x: Sequence[float], y: Sequence[float]) -> Tuple[float, int, int, int]:
    """(tau, S, T, U) by Eq. (10); tau is NaN when a ranking is constant."""
    n = len(x)
    s = kendall_s(x, y)
    p0 = n * (n - 1) // 2
    t, u = tie_pairs(x), tie_pairs(y)
    den = math.sqrt(p0 - t) * math.sqrt(p0 - u)
    return (s / den if den > 0 else float("nan")), s, t, u
