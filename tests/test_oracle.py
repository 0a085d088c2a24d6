"""Pins for the CPU oracle (-m "not gpu").  Each test checks the oracle
against something other than itself: values printed in PAPER.md, closed
forms, theorems, brute force on tiny inputs, or an independent algorithm."""
import math
import os

import numpy as np
import pytest

from oracle.crt import bregman_log2, crt, row_sum_bound, schrijver_lower_log2
from oracle.cryser import per_ryser_nw_c, ryser_nw_partial
from oracle.frontier import per_frontier
from oracle.hybrid import (expand_once, expand_to_leaves, h_per, h_per_node, node_permanent,
                           pre_expand, select_pivot, to_dense, to_rows)
from oracle.kklll import (ROOTS, det_abs2, kklll_all_assignments_mean, kklll_estimate,
                          kklll_trial, mix64, root_index, trial_key)
from oracle.permanent import per_bruteforce, per_ryser, per_ryser_nw_gray
from oracle.schedule import efficiency, lpt, ls, makespan, optimum, order_by_key
from workloads import (dodecahedron, paper_graph, random_3perm, random_3perm_batch,
                       truncated_icosahedron)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _pins():
    d = {}
    with open(os.path.join(GOLD, "paper_pins.txt")) as f:
        for ln in f:
            if ln.strip() and not ln.startswith("#"):
                k, v = ln.split()
                d[k] = v
    return d


# ---------------------------------------------------------------- Eq. (1)
@pytest.mark.parametrize("n", range(1, 8))
def test_bruteforce_closed_forms(n):
    # per(J_n) = n!, per(J_n - I_n) = D_n (derangements: D_n = (n-1)(D_{n-1} + D_{n-2}))
    J = np.ones((n, n), dtype=int)
    assert per_bruteforce(J) == math.factorial(n)
    D = [1, 0]
    for k in range(2, n + 1):
        D.append((k - 1) * (D[k - 1] + D[k - 2]))
    assert per_bruteforce(J - np.eye(n, dtype=int)) == D[n]
    d = np.arange(2, n + 2)
    assert per_bruteforce(np.diag(d)) == int(np.prod(d))


def test_bruteforce_spec_examples():
    assert per_bruteforce([[1, 1, 0], [1, 1, 1], [0, 1, 1]]) == 3
    assert per_bruteforce([[0, 1, 1], [1, 0, 1], [1, 1, 0]]) == 2  # K3: two 3-cycles
    assert per_bruteforce([[1, 2], [3, 4]]) == 10
    assert per_bruteforce([[0, 0], [1, 1]]) == 0


# ---------------------------------------------------------------- R-NW family
def test_ryser_family_equals_bruteforce():
    rng = np.random.default_rng(11)
    for _ in range(150):
        n = int(rng.integers(1, 8))
        a = rng.integers(-3, 4, size=(n, n)) * (rng.random((n, n)) < 0.6)
        b = per_bruteforce(a)
        assert per_ryser(a) == b
        assert per_ryser_nw_gray(a) == b
        assert per_ryser_nw_c(a) == b


def test_ryser_c_partial_ranges_add_up():
    rng = np.random.default_rng(3)
    a = random_3perm(12, rng, weighted=True)
    full = ryser_nw_partial(a, 0, 1 << 11)
    cuts = [0, 7, 300, 1024, 2047, 2048]
    assert sum(ryser_nw_partial(a, cuts[i], cuts[i + 1]) for i in range(5)) == full


def test_ryser_invariances():
    rng = np.random.default_rng(5)
    for _ in range(10):
        a = random_3perm(11, rng, weighted=True)
        p = per_ryser_nw_c(a)
        pr, pc = rng.permutation(11), rng.permutation(11)
        assert per_ryser_nw_c(a[pr][:, pc]) == p
        assert per_ryser_nw_c(a.T) == p
        b = a.copy()
        b[3] *= -5
        assert per_ryser_nw_c(b) == -5 * p


# ---------------------------------------------------------------- Eq. (2)
def test_expand_once_spec_example():
    rows, n = to_rows([[1, 1, 0], [1, 1, 1], [0, 1, 1]])
    assert select_pivot(rows, n) == ("row", 0, 2)
    kids = expand_once(1, rows, n)
    assert len(kids) == 1
    c, m, k = kids[0]
    assert c == 1 and to_dense(m, k) == [[2, 1], [1, 1]]


def test_eq2_identity_all_cases():
    """Sum of coef*per over the children = per(parent) (Eq. (2)),
    for pivots with s = 1..4 on rows and columns, weighted and signed."""
    rng = np.random.default_rng(7)
    seen = set()
    for _ in range(1500):
        n = int(rng.integers(2, 8))
        dens = float(rng.uniform(0.3, 0.95))
        a = rng.integers(-2, 4, size=(n, n)) * (rng.random((n, n)) < dens)
        rows, k = to_rows(a)
        axis, idx, s = select_pivot(rows, k)
        kids = expand_once(3, rows, k)
        if kids is None:
            continue
        seen.add((axis, s))
        tot = sum(c * per_bruteforce(to_dense(m, kk)) for c, m, kk in kids)
        assert tot == 3 * per_bruteforce(a)
        for c, m, kk in kids:
            assert kk == k - 1
    assert {("row", 1), ("row", 2), ("row", 3), ("row", 4), ("col", 1), ("col", 2), ("col", 3)} <= seen


def test_h_per_equals_bruteforce_all_L():
    rng = np.random.default_rng(9)
    for _ in range(120):
        n = int(rng.integers(1, 9))
        a = rng.integers(-2, 4, size=(n, n)) * (rng.random((n, n)) < 0.45)
        b = per_bruteforce(a)
        for L in (2, 3, 5):
            assert h_per(a, L) == b


def test_pre_expand_conservation():
    """SPEC.md:597 style: sum over PH jobs = per(root), every depth."""
    rng = np.random.default_rng(13)
    for _ in range(30):
        n = int(rng.integers(6, 11))
        a = (rng.random((n, n)) < 0.35).astype(int) + np.eye(n, dtype=int)
        ref = per_ryser(a)
        for J in (1, 2, 5, 12):
            jobs = pre_expand(a, jobs_at_least=J)
            assert sum(node_permanent(j) for j in jobs) == ref
            leaves = [l for j in jobs for l in expand_to_leaves(j, 4)]
            assert sum(c * per_ryser(to_dense(m, k)) for c, m, k in leaves) == ref


def test_hybrid_on_3regular_graphs_vs_frontier():
    a = dodecahedron()
    assert h_per(a) == per_frontier(a) == per_ryser_nw_c(a) == 1392
    for a in random_3perm_batch(6, 16, seed=4):
        assert h_per(a) == per_frontier(a) == per_ryser_nw_c(a)


def test_bounds_3regular():
    # Schrijver (4/3)^n <= per(A) <= Bregman 6^(n/3) for 3-regular 0/1 A
    for a in [dodecahedron()] + list(random_3perm_batch(4, 20, seed=8)[:2]):
        n = a.shape[0]
        p = h_per(a)
        assert 2 ** schrijver_lower_log2(n, 3) <= p <= 2 ** bregman_log2(a) * (1 + 1e-12)
        assert p <= row_sum_bound(a)


@pytest.mark.slow
def test_paper_c100_total_by_frontier():
    """PAPER.md:954 (Table T12 Total) by an independent exact method."""
    assert per_frontier(paper_graph("C100")) == int(_pins()["per_C100"])


def test_paper_t12_transcription():
    vals = []
    with open(os.path.join(GOLD, "c100_t12.txt")) as f:
        for ln in f:
            if ln.startswith("#"):
                continue
            k, v = ln.split()
            if k == "Total":
                total = int(v)
            else:
                vals.append(int(v))
    assert len(vals) == 159 and sum(vals) == total == int(_pins()["per_C100"])


def test_c_frontier_pins():
    """oracle/frontier.c: per(C100) = Table T12's Total in C (a few seconds), under
    two row orders; = brute force on small signed matrices (zero rows/columns, n = 0..8); = the
    Python DP on 3-regular n = 20; the closed forms per(J_n) = n!, per(J_n - I_n) = D_n."""
    from oracle.cfrontier import narrow_order, per_frontier_c
    from oracle.frontier import bfs_order
    c100 = paper_graph("C100")
    assert per_frontier_c(c100, bfs_order(c100)) == int(_pins()["per_C100"])
    assert per_frontier_c(c100, narrow_order(c100)) == int(_pins()["per_C100"])
    rng = np.random.default_rng(77)
    for _ in range(60):
        n = int(rng.integers(0, 9))
        a = rng.integers(-3, 4, size=(n, n)) * (rng.random((n, n)) < 0.5)
        order = rng.permutation(n)
        assert per_frontier_c(a, order) == per_bruteforce(a)
    for a in random_3perm_batch(3, 20, seed=5):
        assert per_frontier_c(a, narrow_order(a)) == per_frontier(a)
    for n in (1, 5, 9, 12):
        j = np.ones((n, n), dtype=np.int64)
        d = sum((-1) ** k * math.factorial(n) // math.factorial(k) for k in range(n + 1))
        assert per_frontier_c(j) == math.factorial(n)
        assert per_frontier_c(j - np.eye(n, dtype=np.int64)) == d


@pytest.mark.slow
def test_c60_two_constructions_agree():
    """Appendix C60 and the truncated icosahedron are the
    same graph up to relabelling: equal permanents by the frontier DP; and
    pre-expansion conserves the total (PH Step 4)."""
    from oracle.frontier import bfs_order
    a, b = paper_graph("C60"), truncated_icosahedron()
    pa = per_frontier(a, bfs_order(a))
    assert pa == per_frontier(b, bfs_order(b))
    p = 2 ** bregman_log2(a)
    assert 2 ** schrijver_lower_log2(60, 3) <= pa <= p


# ---------------------------------------------------------------- Kendall tau
def test_kendall_tau_oracle_pins():
    """Eqs. (7)-(10): perfect agreement +1, reversal -1 (the paper's stated
    limits); without ties S = P0 - 2 * inversions (brute-force inversion count); with ties the
    tau-b of scipy.stats.kendalltau (a library routine)."""
    from scipy.stats import kendalltau
    from oracle.stats import kendall_tau_b
    x = list(range(12))
    assert abs(kendall_tau_b(x, x)[0] - 1.0) < 1e-15 and abs(kendall_tau_b(x, x[::-1])[0] + 1.0) < 1e-15
    assert kendall_tau_b(x, x)[1:] == (66, 0, 0)
    rng = np.random.default_rng(3)
    for _ in range(30):
        m = int(rng.integers(2, 40))
        p = rng.permutation(m)
        inv = sum(1 for i in range(m) for j in range(i + 1, m) if p[i] > p[j])
        tau, s, t, u = kendall_tau_b(list(range(m)), list(p))
        assert s == m * (m - 1) // 2 - 2 * inv and t == u == 0
        xs = rng.integers(0, 5, size=m).astype(float)
        ys = rng.integers(0, 4, size=m).astype(float)
        tau, s, t, u = kendall_tau_b(list(xs), list(ys))
        ref = kendalltau(xs, ys).statistic
        assert (math.isnan(tau) and math.isnan(ref)) or abs(tau - ref) < 1e-12


# ---------------------------------------------------------------- KKLLL
def test_kklll_theorem1_exact_expectation():
    """E[X_A] = per(A) (Theorem 1) over all 3^nnz assignments."""
    assert abs(kklll_all_assignments_mean([[1, 1], [1, 1]]) - 2) < 1e-12
    rng = np.random.default_rng(21)
    done = 0
    while done < 6:
        n = int(rng.integers(2, 4))
        a = (rng.random((n, n)) < 0.6).astype(int)
        if a.sum() > 7:
            continue
        assert abs(kklll_all_assignments_mean(a) - per_bruteforce(a)) < 1e-9
        done += 1


def test_kklll_trial_values():
    # all-ones 2x2: |w_a w_d - w_b w_c|^2 in {0, 3}
    for t in range(40):
        x = kklll_trial(np.ones((2, 2)), 5, 0, t)
        assert min(abs(x - 0), abs(x - 3)) < 1e-12
    # identity: product of |w|^2 = 1 up to rounding of sqrt(3)/2
    for t in range(5):
        assert abs(kklll_trial(np.eye(9), 5, 1, t) - 1.0) < 1e-14
    assert kklll_trial(np.zeros((4, 4)), 5, 1, 0) == 0.0


def test_det_abs2_matches_linalg():
    rng = np.random.default_rng(2)
    for n in (1, 2, 5, 17):
        re, im = rng.standard_normal((n, n)), rng.standard_normal((n, n))
        d = np.linalg.det(re + 1j * im)
        assert abs(det_abs2(re, im) - abs(d) ** 2) <= 1e-9 * abs(d) ** 2


def test_kklll_rng_uniform_and_deterministic():
    cnt = [0, 0, 0]
    for t in range(200):
        key = trial_key(7, 3, t)
        for i in range(15):
            cnt[root_index(key, i, (i * 7) % 13)] += 1
    assert all(abs(c - 1000) < 4 * math.sqrt(1000 * 2 / 3) for c in cnt)
    assert mix64(0) == 0 and mix64(1) == 0x5692161D100B05E5  # SplitMix64 finaliser of 1
    assert kklll_estimate(np.ones((4, 4)), 50, 9, 2) == kklll_estimate(np.ones((4, 4)), 50, 9, 2)


def test_kklll_statistical_unbiased():
    a = np.ones((4, 4))
    N = 6000
    xs = [kklll_trial(a, 17, 0, t) for t in range(N)]
    m, s = float(np.mean(xs)), float(np.std(xs, ddof=1))
    assert abs(m - 24) < 4 * s / math.sqrt(N)


# ---------------------------------------------------------------- scheduling
def test_graham_tight_instances():
    a, loads = ls([1, 1, 2], [0, 1, 2], 2)
    assert makespan(loads) == 3 and optimum([1, 1, 2], 2) == 2  # 2 - 1/m
    a, loads = lpt([3, 3, 2, 2, 2], 2)
    assert makespan(loads) == 7 and optimum([3, 3, 2, 2, 2], 2) == 6  # 4/3 - 1/(3m)


def test_graham_bounds_random():
    rng = np.random.default_rng(4)
    for _ in range(150):
        m = int(rng.integers(2, 5))
        p = list(rng.integers(1, 20, size=int(rng.integers(1, 8))).astype(float))
        opt = optimum(p, m)
        assert makespan(ls(p, range(len(p)), m)[1]) <= (2 - 1 / m) * opt + 1e-9
        assert makespan(lpt(p, m)[1]) <= (4 / 3 - 1 / (3 * m)) * opt + 1e-9


def test_efficiency_tables():
    pins = _pins()
    r, e = efficiency(float(pins["table5_T1"]), float(pins["table5_T2"]), 2)
    assert f"{e:.4f}" == pins["table5_eff2"]
    r, e = efficiency(float(pins["table5_T1"]), float(pins["table5_T8"]), 8)
    assert f"{r:.2f}" == pins["table5_ratio8"] and f"{e:.4f}" == pins["table5_eff8"]
    r, e = efficiency(float(pins["table5_T1"]), float(pins["table6_T32"]), 32)
    assert f"{r:.2f}" == pins["table6_ratio32"] and f"{e:.4f}" == pins["table6_eff32"]


def test_order_by_key_ties():
    assert order_by_key([1.0, 3.0, 3.0, 2.0]) == [1, 2, 3, 0]


# ---------------------------------------------------------------- CRT
def test_crt_roundtrip():
    rng = np.random.default_rng(1)
    primes = [2147483647, 2147483629, 2147483587]
    M = primes[0] * primes[1] * primes[2]
    for _ in range(100):
        x = int(rng.integers(-2**62, 2**62)) * int(rng.integers(1, 2**28))
        if abs(x) >= M // 2:
            continue
        assert crt([x % p for p in primes], primes) == x


# ---------------------------------------------------------------- permanental polynomial
def test_permanental_polynomial_oracle_pins():
    """Eq. (11), P(x) = per(xI - A):
      * K_n (A = J - I): c_k = (-1)^(n-k) C(n, k) D_(n-k) (fixed points take x, the rest derange);
      * Lagrange through brute-force values = the brute-force expansion (random signed, n <= 6);
      * C20 (frontier DP values at 21 points): c_20 = 1, c_19 = -trace = 0, c_18 = |E| = 30,
        c_17 = -2 * triangles = 0, c_0 = per(A) = 1392, sum |c_t| = per(I + A)."""
    from oracle.cfrontier import per_frontier_c
    from oracle.permanent import permanental_polynomial, polynomial_from_values
    D = [1, 0]
    for m in range(2, 9):
        D.append((m - 1) * (D[m - 1] + D[m - 2]))
    for n in range(1, 7):
        a = np.ones((n, n), dtype=np.int64) - np.eye(n, dtype=np.int64)
        want = [(-1) ** (n - k) * math.comb(n, k) * D[n - k] for k in range(n + 1)]
        assert permanental_polynomial(a) == want
    rng = np.random.default_rng(41)
    for _ in range(20):
        n = int(rng.integers(1, 7))
        a = rng.integers(-3, 4, size=(n, n)) * (rng.random((n, n)) < 0.6)
        xs = list(range(-(n // 2), n + 1 - n // 2))
        vs = [per_bruteforce(x * np.eye(n, dtype=np.int64) - a) for x in xs]
        assert polynomial_from_values(xs, vs) == permanental_polynomial(a)
    c = c20_polynomial()
    assert c[20] == 1 and c[19] == 0 and c[18] == 30 and c[17] == 0 and c[0] == 1392
    ipa = per_frontier_c(dodecahedron() + np.eye(20, dtype=np.int64))
    assert sum(abs(v) for v in c) == ipa
    assert all((v >= 0) == ((20 - t) % 2 == 0) or v == 0 for t, v in enumerate(c))  # alternating signs


def c20_polynomial():
    """Oracle permanental polynomial of C20: frontier-DP values at x = -10..10, exact Lagrange."""
    from oracle.cfrontier import per_frontier_c
    from oracle.permanent import polynomial_from_values
    a = dodecahedron().astype(np.int64)
    xs = list(range(-10, 11))
    return polynomial_from_values(xs, [per_frontier_c(x * np.eye(20, dtype=np.int64) - a) for x in xs])
