"""Definition-level permanents (test infrastructure only; see oracle/__init__.py).

Matrices are lists of lists of Python ints (or anything convertible).
"""
from __future__ import annotations

from itertools import permutations
from typing import List, Sequence


def _rows(a) -> List[List[int]]:
    return [[int(x) for x in row] for row in a]


def per_bruteforce(a) -> int:
    """Eq. (1): per(A) = sum over all permutations sigma of
    prod_i a[i][sigma(i)].  n <= 10 (factorial cost)."""
    a = _rows(a)
    n = len(a)
    if n > 10:
        raise ValueError("per_bruteforce: n too large")
    total = 0
    for sigma in permutations(range(n)):
        p = 1
        for i in range(n):
            p *= a[i][sigma[i]]
            if p == 0:
                break
        total += p
    return total


def per_ryser(a) -> int:
    """Ryser's inclusion-exclusion formula (the R-NW family named at
    PAPER.md:61-65), written as its plain definition over all 2^n column
    subsets S:  per(A) = (-1)^n sum_S (-1)^{|S|} prod_i sum_{j in S} a_ij.
    No Gray code, no Nijenhuis-Wilf halving.  n <= ~18."""
    a = _rows(a)
    n = len(a)
    if n == 0:
        return 1
    total = 0
    for mask in range(1 << n):
        cols = [j for j in range(n) if (mask >> j) & 1]
        p = 1
        for i in range(n):
            p *= sum(a[i][j] for j in cols)
            if p == 0:
                break
        total += (-1) ** len(cols) * p
    return (-1) ** n * total


def per_ryser_nw_gray(a) -> int:
    """Ryser with the Nijenhuis-Wilf refinement and Gray-code enumeration
    ("R-NW"), exact Python ints, written out directly:

        x_i   = a_{i,n} - (1/2) sum_j a_ij
        per(A) = (-1)^{n-1} * 2 * sum_{S subset of [n-1]} (-1)^{|S|}
                                   prod_i (x_i + sum_{j in S} a_ij)

    evaluated with doubled row sums w_i = 2 x_i + 2 sum_{j in S} a_ij (all
    integers) so per(A) = (-1)^{n-1} 2^{1-n} sum_S (-1)^{|S|} prod_i w_i.
    Subsets are visited in binary-reflected Gray order g(t) = t ^ (t >> 1);
    step t flips column ctz(t).  n <= ~20."""
    a = _rows(a)
    n = len(a)
    if n == 0:
        return 1
    w = [2 * a[i][n - 1] - sum(a[i]) for i in range(n)]
    g = 0
    total = 0
    for t in range(1 << (n - 1)):
        if t:
            j = (t & -t).bit_length() - 1
            g ^= 1 << j
            s = 2 if (g >> j) & 1 else -2
            for i in range(n):
                w[i] += s * a[i][j]
        p = 1
        for i in range(n):
            p *= w[i]
        total += -p if bin(g).count("1") & 1 else p
    num = (-1) ** (n - 1) * total
    den = 1 << (n - 1)
    if num % den:
        raise ArithmeticError("R-NW sum not divisible by 2^(n-1)")
    return num // den


def per_dense_small(a) -> int:
    """per of an order <= 2 matrix written out (H_per leaves with L = 2)."""
    a = _rows(a)
    n = len(a)
    if n == 0:
        return 1
    if n == 1:
        return a[0][0]
    if n == 2:
        return a[0][0] * a[1][1] + a[0][1] * a[1][0]
    raise ValueError("order > 2")


def transpose(a: Sequence[Sequence[int]]) -> List[List[int]]:
    return [list(r) for r in zip(*a)] if len(a) else []


def permanental_polynomial(a) -> list:
    """Coefficients [c_0..c_n] of per(xI - A) (Eq. (11)) by Eq. (1) itself:
    every permutation sigma contributes prod_i (x [sigma(i) = i] - a_{i sigma(i)}), a polynomial
    in x multiplied out term by term.  Brute force (n <= 8)."""
    from itertools import permutations
    a = [[int(v) for v in row] for row in a]
    n = len(a)
    total = [0] * (n + 1)
    for sigma in permutations(range(n)):
        poly = [1]  # coefficients of the running product
        for i in range(n):
            j = sigma[i]
            f = [-a[i][j], 1 if i == j else 0]  # x [i == j] - a_ij
            nxt = [0] * (len(poly) + 1)
            for d, c in enumerate(poly):
                nxt[d] += c * f[0]
                nxt[d + 1] += c * f[1]
            poly = nxt
        for d, c in enumerate(poly):
            total[d] += c
    return total


def polynomial_from_values(xs, vs) -> list:
    """Exact coefficients of the polynomial of degree < len(xs) through (xs[j], vs[j]), by
    Lagrange's formula in rational arithmetic (fractions.Fraction)."""
    from fractions import Fraction
    m = len(xs)
    coef = [Fraction(0)] * m
    for j in range(m):
        num = [Fraction(1)]  # prod_{i != j} (x - x_i)
        den = Fraction(1)
        for i in range(m):
            if i == j:
                continue
            num = [Fraction(0)] + num
            for d in range(len(num) - 1):
                num[d] -= xs[i] * num[d + 1]
            den *= xs[j] - xs[i]
        for d in range(m):
            coef[d] += vs[j] * num[d] / den
    out = []
    for c in coef:
        if c.denominator != 1:
            raise ArithmeticError("non-integer coefficient")
        out.append(int(c))
    return out
