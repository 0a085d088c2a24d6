"""Eq. (2) expansion, Algorithm H_per and Algorithm PH Step 2 (test
infrastructure only; see oracle/__init__.py).

A node is (coef, rows, n): the matrix of order n is stored as a list of n
sparse rows {column: nonzero value}; the node contributes coef * per(matrix).

Readings of the paper taken here (all listed in DESIGN.md §2):
  R1  s = minimal number of nonzeros over all 2n lines, counted on the
      nonzero pattern.
  R2  Pivot tie-break (paper silent): rows before columns, lowest index first;
      a column pivot is handled as a row pivot of the transpose
      (per(A) = per(A^T)).
  R3  The pivot line's nonzeros, in ascending position p0<p1<p2<p3, are
      Eq. (2)'s a, b, c, d.  Child A1 = merge of p0,p1:
      column p0 := a*col(p1) + b*col(p0), column p1 and the pivot row deleted,
      other columns keep their relative order (Eq. (2) writes the merged
      column first; per() is invariant under column order).  For s = 4,
      A2 = merge of p2,p3 the same way.  For s = 3, A2 is the cofactor
      c * minor(row, p2) and for s = 1 the only child is a * minor(row, p0)
      (Eq. (2) with the missing scalars equal to 0 leaves the scalar on a
      single column; we carry it in coef instead).  s = 2 has one child
      (A2 has a zero column).
  R4  Children with a zero row or column have per = 0 and are dropped.
  R5  H_per leaf rule: expand while n > L and s < 5, else evaluate the leaf
      with R-NW (PAPER.md:133-136 has L = 2; the leaf-order threshold L is
      the build's parameter).
  R6  PH Step 2 expands level by level in natural order
      (child A1 before A2, parents in order).  It stops when the job count
      reaches `jobs_at_least` or the order reaches `job_order`; nodes with
      s >= 5 stop early and are appended after the level's nodes.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

from .permanent import per_dense_small, per_ryser

Rows = List[Dict[int, int]]
Node = Tuple[int, Rows, int]  # (coef, rows, n)


# ---------------------------------------------------------------------------
# conversions
# ---------------------------------------------------------------------------
def to_rows(a) -> Tuple[Rows, int]:
    n = len(a)
    rows = []
    for i in range(n):
        if len(a[i]) != n:
            raise ValueError("matrix must be square")
        rows.append({j: int(a[i][j]) for j in range(n) if int(a[i][j]) != 0})
    return rows, n


def to_dense(rows: Rows, n: int) -> List[List[int]]:
    out = [[0] * n for _ in range(n)]
    for i, r in enumerate(rows):
        for j, x in r.items():
            out[i][j] = x
    return out


def transpose_rows(rows: Rows, n: int) -> Rows:
    t: Rows = [dict() for _ in range(n)]
    for i, r in enumerate(rows):
        for j, x in r.items():
            t[j][i] = x
    return t


# ---------------------------------------------------------------------------
# Step 1 of H_per: the pivot line
# ---------------------------------------------------------------------------
def line_counts(rows: Rows, n: int) -> Tuple[List[int], List[int]]:
    rc = [len(r) for r in rows]
    cc = [0] * n
    for r in rows:
        for j in r:
            cc[j] += 1
    return rc, cc


def select_pivot(rows: Rows, n: int) -> Tuple[str, int, int]:
    """Algorithm H_per Step 1 with reading R1/R2.
    Returns (axis, index, s) with axis in {"row", "col"}."""
    rc, cc = line_counts(rows, n)
    best = ("row", 0, rc[0]) if n else ("row", 0, 0)
    for i in range(n):
        if rc[i] < best[2]:
            best = ("row", i, rc[i])
    for j in range(n):
        if cc[j] < best[2]:
            best = ("col", j, cc[j])
    return best


# ---------------------------------------------------------------------------
# Eq. (2)
# ---------------------------------------------------------------------------
def _merge(rows: Rows, r: int, keep: int, drop: int, alpha: int, beta: int) -> Rows:
    """Delete row r; column keep := alpha*col(drop) + beta*col(keep);
    delete column drop (keep < drop)."""
    out: Rows = []
    for i, row in enumerate(rows):
        if i == r:
            continue
        new: Dict[int, int] = {}
        for j, x in row.items():
            if j == keep or j == drop:
                continue
            new[j - (1 if j > drop else 0)] = x
        val = alpha * row.get(drop, 0) + beta * row.get(keep, 0)
        if val != 0:
            new[keep] = val
        out.append(new)
    return out


def _minor(rows: Rows, r: int, c: int) -> Rows:
    out: Rows = []
    for i, row in enumerate(rows):
        if i == r:
            continue
        out.append({(j - (1 if j > c else 0)): x for j, x in row.items() if j != c})
    return out


def has_zero_line(rows: Rows, n: int) -> bool:
    if any(len(r) == 0 for r in rows):
        return True
    seen = set()
    for r in rows:
        seen.update(r.keys())
    return len(seen) != n


def expand_row(coef: int, rows: Rows, n: int, r: int) -> List[Node]:
    """Eq. (2) on pivot row r with s = nnz(row r) <= 4,
    readings R3/R4.  Returns the surviving children in natural order."""
    pos = sorted(rows[r].keys())
    s = len(pos)
    if s > 4:
        raise ValueError("Eq. (2) with per(A3) = 0 needs s <= 4")
    vals = [rows[r][p] for p in pos]
    kids: List[Node] = []
    if s == 0:
        return []
    if s == 1:
        kids.append((coef * vals[0], _minor(rows, r, pos[0]), n - 1))
    else:
        a, b = vals[0], vals[1]
        kids.append((coef, _merge(rows, r, pos[0], pos[1], a, b), n - 1))
        if s == 3:
            kids.append((coef * vals[2], _minor(rows, r, pos[2]), n - 1))
        elif s == 4:
            c, d = vals[2], vals[3]
            kids.append((coef, _merge(rows, r, pos[2], pos[3], c, d), n - 1))
    return [k for k in kids if not has_zero_line(k[1], k[2])]


def expand_once(coef: int, rows: Rows, n: int) -> Optional[List[Node]]:
    """One H_per split of a node: None if s >= 5 (not expandable),
    [] if s == 0 (per = 0), else the 1 or 2 children (R1-R4)."""
    axis, idx, s = select_pivot(rows, n)
    if s >= 5:
        return None
    if s == 0:
        return []
    if axis == "row":
        return expand_row(coef, rows, n, idx)
    kids = expand_row(coef, transpose_rows(rows, n), n, idx)
    return [(c, transpose_rows(m, k), k) for (c, m, k) in kids]


# ---------------------------------------------------------------------------
# Algorithm H_per
# ---------------------------------------------------------------------------
def leaf_permanent(rows: Rows, n: int) -> int:
    """R-NW(A) of H_per Step 2: for order <= 2 written out, else Ryser."""
    d = to_dense(rows, n)
    if n <= 2:
        return per_dense_small(d)
    return per_ryser(d)


def h_per(a, L: int = 2) -> int:
    """Algorithm H_per with leaf threshold L (R5)."""
    rows, n = to_rows(a)
    return h_per_node(1, rows, n, L)


def h_per_node(coef: int, rows: Rows, n: int, L: int = 2) -> int:
    stack: List[Node] = [(coef, rows, n)]
    total = 0
    while stack:
        c, m, k = stack.pop()
        if k == 0:
            total += c
            continue
        kids = expand_once(c, m, k) if k > L else None
        if kids is None:
            total += c * leaf_permanent(m, k)
        else:
            stack.extend(kids)
    return total


# ---------------------------------------------------------------------------
# Algorithm PH Step 2 and the continuation of each job to its leaves
# ---------------------------------------------------------------------------
def pre_expand(a, jobs_at_least: int = 1, job_order: int = 1) -> List[Node]:
    """PH Step 2, reading R6: breadth-first levels in
    natural order until len(jobs) >= jobs_at_least or order <= job_order."""
    rows, n = to_rows(a)
    level: List[Node] = [(1, rows, n)]
    early: List[Node] = []
    order = n
    if has_zero_line(rows, n):
        return []
    while level and len(level) + len(early) < jobs_at_least and order > job_order:
        nxt: List[Node] = []
        for c, m, k in level:
            kids = expand_once(c, m, k)
            if kids is None:
                early.append((c, m, k))
            else:
                nxt.extend(kids)
        level = nxt
        order -= 1
    return level + early


def expand_to_leaves(node: Node, L: int) -> List[Node]:
    """H_per's recursion applied breadth-first to one job until every node has
    order <= L or s >= 5 (R5, R6).  Level leaves first, then early leaves."""
    level: List[Node] = [node]
    early: List[Node] = []
    order = node[2]
    while level and order > L:
        nxt: List[Node] = []
        for c, m, k in level:
            kids = expand_once(c, m, k)
            if kids is None:
                early.append((c, m, k))
            else:
                nxt.extend(kids)
        level = nxt
        order -= 1
    return level + early


def node_permanent(node: Node, L: int = 2) -> int:
    c, m, k = node
    return h_per_node(c, m, k, L)
