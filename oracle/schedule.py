"""Parallel machine scheduling and the improved Step 3
 — test infrastructure only.

  ls(p, order, m)   Algorithm LS: jobs in the given order, each to the
                    currently least-loaded machine (tie -> lowest machine id).
  lpt(p, m)         Algorithm LPT: non-increasing p, ties -> lower job id, then LS.
  by_key(keys, ...) the order used by PH's Step 3: non-increasing key, ties ->
                    lower job id (keys = KKLLL estimates for the improved
                    Step 3).
  optimum(p, m)     exhaustive minimum makespan (<= 10 jobs), for the Graham
                    bounds 2 - 1/m (LS) and 4/3 - 1/(3m) (LPT).
  efficiency(T1, Tm, m)  accelerated ratio T1/Tm and efficiency T1/(m Tm),
                    Tables 5-10.
"""
from __future__ import annotations

from itertools import product
from typing import List, Sequence, Tuple


def order_by_key(keys: Sequence[float]) -> List[int]:
    return sorted(range(len(keys)), key=lambda j: (-keys[j], j))


def ls(p: Sequence[float], order: Sequence[int], m: int) -> Tuple[List[int], List[float]]:
    """Returns (machine of each job, machine loads)."""
    loads = [0.0] * m
    assign = [-1] * len(p)
    for j in order:
        k = min(range(m), key=lambda t: (loads[t], t))
        assign[j] = k
        loads[k] += p[j]
    return assign, loads


def lpt(p: Sequence[float], m: int):
    return ls(p, order_by_key(p), m)


def makespan(loads: Sequence[float]) -> float:
    return max(loads) if loads else 0.0


def optimum(p: Sequence[float], m: int) -> float:
    if len(p) > 10:
        raise ValueError("too many jobs")
    best = float("inf")
    for a in product(range(m), repeat=len(p)):
        if a and a[0] != 0:
            continue  # machine symmetry
        loads = [0.0] * m
        for j, k in enumerate(a):
            loads[k] += p[j]
        best = min(best, max(loads))
    return best if p else 0.0


def efficiency(T1: float, Tm: float, m: int) -> Tuple[float, float]:
    if T1 <= 0 or Tm <= 0:
        raise ValueError("times must be positive")
    r = T1 / Tm
    return r, r / m
