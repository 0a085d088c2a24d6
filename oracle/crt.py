"""Chinese remaindering and permanent bounds — test infrastructure only.

crt(residues, primes): the unique x with x = r_i (mod p_i) in the symmetric
range -M/2 < x <= M/2, M = prod p_i, written as the textbook sum
x = sum_i r_i * M_i * (M_i^{-1} mod p_i)  (mod M).

Bounds used to size the prime set:
  row_sum_bound(A) = prod_i sum_j |a_ij|  >= |per(A)|  (expand the product)
  bregman(A)       = prod_i (r_i!)^{1/r_i} >= per(A) for 0/1 A (Bregman 1973)
"""
from __future__ import annotations

import math
from typing import Sequence


def crt(residues: Sequence[int], primes: Sequence[int]) -> int:
    M = 1
    for p in primes:
        M *= p
    x = 0
    for r, p in zip(residues, primes):
        Mi = M // p
        x += int(r) * Mi * pow(Mi, -1, p)
    x %= M
    if x > M // 2:
        x -= M
    return x


def row_sum_bound(a) -> int:
    b = 1
    for row in a:
        b *= sum(abs(int(x)) for x in row)
    return b


def bregman_log2(a) -> float:
    s = 0.0
    for row in a:
        r = sum(1 for x in row if int(x) != 0)
        if r == 0:
            return float("-inf")
        s += math.lgamma(r + 1) / r / math.log(2)
    return s


def schrijver_lower_log2(n: int, k: int) -> float:
    """Schrijver (1998): a k-regular bipartite graph on 2n vertices has at
    least ((k-1)^{k-1} / k^{k-2})^n perfect matchings."""
    return n * ((k - 1) * math.log2(k - 1) - (k - 2) * math.log2(k))
