"""Graph and matrix builders for the seeded synthetic workloads.

Nothing here evaluates a permanent; these are inputs only (see __init__.py).
Every random choice is drawn from numpy's PCG64 seeded explicitly, so a
(seed, index) pair always yields the same matrix on every machine.
"""
from __future__ import annotations

import os
from collections import deque
from typing import Dict, List, Sequence, Tuple

import numpy as np

_DATA = os.path.join(os.path.dirname(__file__), "data")


# ---------------------------------------------------------------------------
# adjacency helpers
# ---------------------------------------------------------------------------
def adjacency_matrix(n: int, edges) -> np.ndarray:
    """0/1 symmetric int64 adjacency matrix of an undirected simple graph
    (0-based vertex ids)."""
    a = np.zeros((n, n), dtype=np.int64)
    for u, v in edges:
        if u == v:
            raise ValueError("self loop")
        a[u, v] = 1
        a[v, u] = 1
    return a


def _edges_from_adjlists(adj: Sequence[Sequence[int]]) -> List[Tuple[int, int]]:
    e = set()
    for u, nb in enumerate(adj):
        for v in nb:
            e.add((min(u, v), max(u, v)))
    return sorted(e)


# ---------------------------------------------------------------------------
# paper data (PAPER.md Appendix)
# ---------------------------------------------------------------------------
def paper_graph(name: str) -> np.ndarray:
    """Adjacency matrix of the appendix fullerene `name` in {"C60", "C100"}.

    Transcribed from PAPER.md:624-647 (C100) and PAPER.md:653-668 (C60), the
    MATLAB tables `D` with `A(k, D(k,:)) = 1`.  The data
    files list, for vertex k = 1..n, its three neighbours (1-based)."""
    fn = {"C60": "c60.adj", "C100": "c100.adj"}.get(name)
    if fn is None:
        raise KeyError(f"unknown builtin dataset {name!r}")
    rows = []
    with open(os.path.join(_DATA, fn)) as f:
        for ln in f:
            ln = ln.strip()
            if not ln or ln.startswith("#"):
                continue
            rows.append([int(x) for x in ln.split()])
    n = len(rows)
    a = np.zeros((n, n), dtype=np.int64)
    for k, nb in enumerate(rows):
        for v in nb:
            if not 1 <= v <= n:
                raise ValueError("index out of range")
            a[k, v - 1] = 1
    return a


# ---------------------------------------------------------------------------
# closed-form polyhedra
# ---------------------------------------------------------------------------
def dodecahedron() -> np.ndarray:
    """C20 (configs[0]): outer 5-cycle o_k, middle 10-cycle m_j, inner 5-cycle
    i_k, with spokes o_k - m_{2k} and i_k - m_{2k+1} (generalised Petersen
    graph GP(10,2)); exactly 3 ones per row and column."""
    o = lambda k: k % 5            # noqa: E731
    m = lambda j: 5 + (j % 10)     # noqa: E731
    i = lambda k: 15 + (k % 5)     # noqa: E731
    e = []
    for k in range(5):
        e.append((o(k), o(k + 1)))
        e.append((i(k), i(k + 1)))
        e.append((o(k), m(2 * k)))
        e.append((i(k), m(2 * k + 1)))
    for j in range(10):
        e.append((m(j), m(j + 1)))
    return adjacency_matrix(20, e)


def icosahedron() -> List[List[int]]:
    """Icosahedron as adjacency lists: top T=0, upper pentagon U_k=1+k, lower
    pentagon L_k=6+k (antiprism U_k-L_k, U_k-L_{k+1}), bottom B=11."""
    adj = [set() for _ in range(12)]

    def add(u, v):
        adj[u].add(v)
        adj[v].add(u)

    for k in range(5):
        U, U1 = 1 + k, 1 + (k + 1) % 5
        L, L1 = 6 + k, 6 + (k + 1) % 5
        add(0, U)
        add(U, U1)
        add(U, L)
        add(U, L1)
        add(L, L1)
        add(11, L)
    return [sorted(s) for s in adj]


def truncated_icosahedron() -> np.ndarray:
    """C60 (configs[2]): the truncation of the icosahedron.  Vertex (u,v) for
    each directed edge u->v of the icosahedron; (u,v) ~ (v,u) (the cut edge)
    and (u,v) ~ (u,w) when v ~ w (the pentagon that replaces vertex u)."""
    ico = icosahedron()
    ids: Dict[Tuple[int, int], int] = {}
    for u in range(12):
        for v in ico[u]:
            ids[(u, v)] = len(ids)
    e = []
    for (u, v), a in ids.items():
        b = ids[(v, u)]
        if a < b:
            e.append((a, b))
        for w in ico[u]:
            if w > v and w in ico[v]:
                e.append((a, ids[(u, w)]))
    return adjacency_matrix(60, e)


# ---------------------------------------------------------------------------
# random 3-regular bipartite matrices (configs[1], configs[4])
# ---------------------------------------------------------------------------
def random_3perm(n: int, rng: np.random.Generator, weighted: bool = False,
                 wmax: int = 7) -> np.ndarray:
    """Sum of 3 random n x n permutation matrices, each redrawn until it is
    disjoint from the previous ones, so every row and column has exactly 3
    nonzeros.  If `weighted`, each nonzero is then replaced by an independent
    uniform integer in [1, wmax] (drawn row-major, one per nonzero)."""
    perms: List[np.ndarray] = []
    for _ in range(3):
        while True:
            p = rng.permutation(n)
            if all(not np.any(p == q) for q in perms):
                perms.append(p)
                break
    a = np.zeros((n, n), dtype=np.int64)
    for p in perms:
        a[np.arange(n), p] = 1
    if weighted:
        r, c = np.nonzero(a)
        a[r, c] = rng.integers(1, wmax + 1, size=len(r))
    return a


def random_3perm_batch(count: int = 256, n: int = 24, seed: int = 2024,
                       wmax: int = 7) -> np.ndarray:
    """configs[1]: `count` matrices; the first half 0/1, the second half with
    nonzeros uniform in [1, wmax].  Matrix i uses PCG64([seed, i])."""
    out = np.zeros((count, n, n), dtype=np.int64)
    for i in range(count):
        rng = np.random.Generator(np.random.PCG64([seed, i]))
        out[i] = random_3perm(n, rng, weighted=(i >= count // 2), wmax=wmax)
    return out


def random_sparse01(n: int, nnz: int, rng: np.random.Generator) -> np.ndarray:
    """Uniformly random 0/1 n x n matrix with exactly `nnz` ones (test input)."""
    a = np.zeros(n * n, dtype=np.int64)
    a[rng.choice(n * n, size=nnz, replace=False)] = 1
    return a.reshape(n, n)


# ---------------------------------------------------------------------------
# fullerenes from face spirals (configs[3], configs[4])
# ---------------------------------------------------------------------------
class SpiralFail(Exception):
    pass


def spiral_windup(spiral: Sequence[int]):
    """Wind up a face spiral into a planar triangulation (the dual of the
    fullerene).  `spiral[k]` is the size (5 or 6) of face k = the degree of
    dual vertex k.  Each new vertex k is attached to the outer-boundary edge
    (newest, oldest); boundary vertices whose valence is used up are closed
    off by joining their two boundary neighbours.  Returns the list of
    triangles, or raises SpiralFail if the spiral does not close."""
    F = len(spiral)
    deg = list(spiral)
    adj = [set() for _ in range(F)]
    tris: List[Tuple[int, int, int]] = []

    def connect(u, v):
        if u == v or v in adj[u]:
            raise SpiralFail("multi-edge")
        adj[u].add(v)
        adj[v].add(u)
        if len(adj[u]) > deg[u] or len(adj[v]) > deg[v]:
            raise SpiralFail("valence")

    def rem(v):
        return deg[v] - len(adj[v])

    if F < 4:
        raise SpiralFail("too small")
    connect(0, 1)
    bnd = deque([0, 1])
    for k in range(2, F):
        newest, oldest = bnd[-1], bnd[0]
        connect(k, newest)
        connect(k, oldest)
        tris.append((newest, oldest, k))
        bnd.append(k)
        changed = True
        while changed and len(bnd) > 3:
            changed = False
            if rem(bnd[0]) == 0:
                b0 = bnd.popleft()
                connect(k, bnd[0])
                tris.append((b0, bnd[0], k))
                changed = True
                continue
            if rem(bnd[-2]) == 0:
                bm = bnd[-2]
                del bnd[-2]
                connect(k, bnd[-2])
                tris.append((bnd[-2], bm, k))
                changed = True
    if len(bnd) != 3 or any(rem(v) != 0 for v in bnd):
        raise SpiralFail("open boundary")
    tris.append(tuple(bnd))
    if len(tris) != 2 * F - 4 or any(rem(v) != 0 for v in range(F)):
        raise SpiralFail("not a triangulation")
    return tris


def _dual_of_triangles(tris) -> np.ndarray:
    owner: Dict[Tuple[int, int], List[int]] = {}
    for t, (a, b, c) in enumerate(tris):
        for u, v in ((a, b), (b, c), (c, a)):
            owner.setdefault((min(u, v), max(u, v)), []).append(t)
    e = []
    for key, ts in owner.items():
        if len(ts) != 2:
            raise SpiralFail("edge not shared by two triangles")
        e.append((ts[0], ts[1]))
    g = adjacency_matrix(len(tris), e)
    if not np.all(g.sum(1) == 3):
        raise SpiralFail("dual not cubic")
    return g


def spiral_fullerene(pentagons: Sequence[int], n: int) -> np.ndarray:
    """Fullerene with n atoms from the 0-based positions of its 12 pentagons in
    the face spiral of F = n/2 + 2 faces."""
    F = n // 2 + 2
    if n % 2 or len(set(pentagons)) != 12:
        raise ValueError("need even n and 12 distinct pentagon positions")
    spiral = [6] * F
    for p in pentagons:
        spiral[p] = 5
    return _dual_of_triangles(spiral_windup(spiral))


def random_fullerene(n: int, seed: int, isomer: int = 0, max_tries: int = 2_000_000):
    """configs[3]/[4]: a seeded fullerene isomer with n atoms: random pentagon
    positions in the face spiral (PCG64([seed, n, isomer])), rejected until the
    spiral closes.  Returns (adjacency matrix, pentagon positions)."""
    F = n // 2 + 2
    rng = np.random.Generator(np.random.PCG64([seed, n, isomer]))
    for _ in range(max_tries):
        pos = sorted(int(x) for x in rng.choice(F, size=12, replace=False))
        try:
            return spiral_fullerene(pos, n), pos
        except SpiralFail:
            continue
    raise RuntimeError("no closing spiral found")


# ---------------------------------------------------------------------------
# face census (validation of inputs only)
# ---------------------------------------------------------------------------
def face_cycles(a: np.ndarray, length: int) -> int:
    """Number of induced cycles of the given length in the graph (for a
    fullerene, length 5 counts pentagons)."""
    n = a.shape[0]
    nb = [list(np.nonzero(a[i])[0]) for i in range(n)]
    found = set()

    def dfs(start, path, seen):
        u = path[-1]
        if len(path) == length:
            if start in nb[u]:
                cyc = tuple(path)
                # induced: no chords
                ok = all((cyc[j] not in nb[cyc[i]]) for i in range(length)
                         for j in range(i + 2, length) if not (i == 0 and j == length - 1))
                if ok:
                    k = min(range(length), key=lambda t: cyc[t])
                    r = cyc[k:] + cyc[:k]
                    if r[1] > r[-1]:
                        r = (r[0],) + tuple(reversed(r[1:]))
                    found.add(r)
            return
        for v in nb[u]:
            if v > start and v not in seen:
                seen.add(v)
                path.append(v)
                dfs(start, path, seen)
                path.pop()
                seen.discard(v)

    for s in range(n):
        dfs(s, [s], {s})
    return len(found)
