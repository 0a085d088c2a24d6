"""Row-frontier dynamic programme for per(A) (test infrastructure only).

Not a method of the paper: an independent exact algorithm used to pin the
paper's printed total per(C100) = 149364113290700 (Table T12)
and to cross-check H_per on graphs too large for brute force.

per(A) = sum over perfect matchings rows -> columns.  Process rows in order;
the state is the set of columns already used that are still "open" (some
later row has a nonzero there).  A column whose last nonzero row has been
processed must be used by then, otherwise the partial assignment can never be
completed and the state is discarded.  Exact Python integers.
"""
from __future__ import annotations

from typing import Dict, Sequence


def per_frontier(a, row_order: Sequence[int] = None) -> int:
    n = len(a)
    rows = list(range(n)) if row_order is None else list(row_order)
    if sorted(rows) != list(range(n)):
        raise ValueError("row_order must be a permutation")
    nz = [[(j, int(a[i][j])) for j in range(n) if int(a[i][j]) != 0] for i in range(n)]
    last = {}
    for step, i in enumerate(rows):
        for j, _ in nz[i]:
            last[j] = step
    if len(last) != n:
        return 0  # a zero column
    closes = [[] for _ in range(n)]
    for j, step in last.items():
        closes[step].append(j)
    states: Dict[int, int] = {0: 1}
    for step, i in enumerate(rows):
        nxt: Dict[int, int] = {}
        for used, val in states.items():
            for j, x in nz[i]:
                bit = 1 << j
                if used & bit:
                    continue
                key = used | bit
                nxt[key] = nxt.get(key, 0) + val * x
        for j in closes[step]:
            bit = 1 << j
            nxt = {k & ~bit: v for k, v in nxt.items() if k & bit}
        states = nxt
        if not states:
            return 0
    return sum(states.values())


def bfs_order(a, start: int = 0):
    """Breadth-first row order of a symmetric pattern (keeps the frontier
    narrow on fullerene graphs)."""
    n = len(a)
    seen = [False] * n
    order = []
    for s in [start] + list(range(n)):
        if seen[s]:
            continue
        seen[s] = True
        q = [s]
        while q:
            u = q.pop(0)
            order.append(u)
            for v in range(n):
                if a[u][v] and not seen[v]:
                    seen[v] = True
                    q.append(v)
    return order
