"""CPU-only checks of the C-ABI library (-m "not gpu"): it loads, exports every
symbol include/sperm.h declares, and its host-side functions (CRT, scheduler)
agree with the oracle.  No kernel is launched here."""
import math
import os
import re

import numpy as np
import pytest

import paper_1112_6072_b200 as P
from paper_1112_6072_b200 import sperm as S
from oracle.crt import crt as oracle_crt
from oracle.schedule import lpt, ls, makespan, order_by_key

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "sperm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sperm_\w+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    L = P.lib()
    names = _header_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(S.SYMBOLS), "binding and header disagree"


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_1112_6072_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.findall(r"(?:import|from)\s+(\w+)", src), f


def test_primes():
    ps = P.primes(8)
    assert ps == sorted(ps, reverse=True) and len(set(ps)) == 8
    for p in ps:
        assert 2**30 < p < 2**31
        assert all(p % d for d in range(2, int(math.isqrt(p)) + 1, 1 if p < 100 else 2) if d == 2 or d % 2)
    assert P.sperm_prime(8) == 0 and P.sperm_prime(-1) == 0


def test_crt_matches_oracle():
    rng = np.random.default_rng(5)
    for k in range(1, 9):
        ps = P.primes(k)
        M = math.prod(ps)
        for _ in range(40):
            x = int(rng.integers(-2**62, 2**62)) * int(rng.integers(0, 2**60)) ** (k // 2 + 1) % M
            if x > M // 2:
                x -= M
            res = [x % p for p in ps]
            assert P.sperm_crt(res, k) == x == oracle_crt(res, ps)
        # extremes of the symmetric range
        for x in (M // 2, -(M // 2) + (M % 2 == 0), 0, 1, -1):
            assert P.sperm_crt([x % p for p in ps], k) == x


def test_crt_bad_args():
    with pytest.raises(S.SpermError):
        S.sperm_crt([1, 2, 3], 0)


@pytest.mark.parametrize("m", [1, 2, 3, 8, 32])
def test_schedule_lpt_matches_oracle(m):
    rng = np.random.default_rng(m)
    for _ in range(20):
        w = list(rng.integers(1, 50, size=int(rng.integers(1, 60))).astype(float))
        w[0] = w[-1]  # ties
        mach, order, loads = P.sperm_schedule(w, m, "estimate")
        assign, oloads = lpt(w, m)
        assert list(order) == order_by_key(w)
        assert list(mach) == assign
        assert np.allclose(loads, oloads)


def test_schedule_natural_is_ls():
    w = [5.0, 1.0, 1.0, 2.0, 7.0, 3.0]
    mach, order, loads = P.sperm_schedule(w, 3, "natural")
    assign, oloads = ls(w, range(len(w)), 3)
    assert list(order) == list(range(6)) and list(mach) == assign and np.allclose(loads, oloads)


def test_schedule_graham_tight():
    _, _, loads = P.sperm_schedule([3, 3, 2, 2, 2], 2, "estimate")
    assert makespan(list(loads)) == 7  # 4/3 - 1/(3m) instance
    _, _, loads = P.sperm_schedule([1, 1, 2], 2, "natural")
    assert makespan(list(loads)) == 3  # 2 - 1/m instance


def test_schedule_random_is_permutation_and_seeded():
    w = list(range(100))
    _, o1, _ = P.sperm_schedule(w, 4, "random", seed=3)
    _, o2, _ = P.sperm_schedule(w, 4, "random", seed=3)
    _, o3, _ = P.sperm_schedule(w, 4, "random", seed=4)
    assert sorted(o1) == w and list(o1) == list(o2) and list(o1) != list(o3)


def test_schedule_empty():
    mach, order, loads = P.sperm_schedule([], 4)
    assert len(mach) == 0 and list(loads) == [0, 0, 0, 0]


def test_rnw_terms():
    assert P.sperm_rnw_terms(24, 256) == 256 * 2**23
    assert P.sperm_rnw_terms(1, 3) == 3


def test_cuda_entry_points_fail_loudly_without_device():
    """No GPU here: a compute call must raise, never fall back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(TypeError):
        P.sperm_permanent(torch.zeros((1, 3, 3), dtype=torch.int32))


def test_bound_primes_sufficient_and_tight():
    """sperm_bound_primes: product of the primes > 2 * bound (oracle.crt bounds, exact ints),
    and one prime fewer would not cover the bound."""
    from oracle.crt import bregman_log2, row_sum_bound
    from workloads import dodecahedron, paper_graph, random_3perm_batch, truncated_icosahedron
    rng = np.random.default_rng(3)
    mats = [dodecahedron(), truncated_icosahedron(), paper_graph("C100"), np.ones((7, 7), int),
            np.zeros((3, 3), int)] + list(random_3perm_batch(256, 24, seed=2024)[[0, 1, 130, 131]])
    mats += [rng.integers(-9, 10, size=(10, 10)) for _ in range(5)]
    for a in mats:
        k = P.sperm_bound_primes(a)
        b = min(row_sum_bound(a), row_sum_bound(np.asarray(a).T))
        lb = math.log2(b) if b > 0 else -1
        if np.isin(a, (0, 1)).all() and b > 0:
            lb = min(lb, bregman_log2(a), bregman_log2(np.asarray(a).T))
        M = math.prod(P.primes(k))
        assert math.log2(M) > lb + 1
        if k > 1:
            assert math.log2(math.prod(P.primes(k - 1))) <= lb + 1 + 1e-6
    # C100: per = 149364113290700 (Table T12) < 2^48 needs 2 primes; Bregman 6^(100/3) -> 3
    assert P.sperm_bound_primes(paper_graph("C100")) == 3
    assert P.sperm_bound_primes(truncated_icosahedron()) == 2


def test_kendall_tau_matches_oracle_definition():
    """sperm_kendall_tau (host C++, O(m log m)) = the O(m^2) definition of Eqs. (7)-(10)
    (oracle/stats.py): S, T, U exactly and tau to the last bit of the same formula, on
    random keys with heavy ties, all-distinct keys, constant keys and tiny inputs."""
    import math
    from oracle.stats import kendall_tau_b
    rng = np.random.default_rng(8)
    cases = [([], []), ([1.0], [2.0]), ([1.0, 1.0], [2.0, 3.0]), ([3.0, 1.0, 2.0], [1.0, 2.0, 3.0])]
    for _ in range(60):
        m = int(rng.integers(2, 300))
        k = int(rng.integers(1, 12))
        cases.append((list(rng.integers(0, k, size=m).astype(float)), list(rng.integers(0, k + 3, size=m).astype(float))))
        cases.append((list(rng.random(m)), list(rng.random(m))))
    for x, y in cases:
        got, (s, t, u, p0) = S.sperm_kendall_tau(x, y, return_counts=True)
        m = len(x)
        if m < 2:
            assert s == t == u == p0 == 0 and math.isnan(got)
            continue
        tau, s0, t0, u0 = kendall_tau_b(x, y)
        assert (s, t, u, p0) == (s0, t0, u0, m * (m - 1) // 2)
        assert (math.isnan(got) and math.isnan(tau)) or got == tau


def test_list_schedule_matches_oracle_ls():
    """sperm_list_schedule = oracle.schedule.ls (Algorithm LS) on random
    costs and orders, ties included; efficiency = sum / (m * makespan)."""
    rng = np.random.default_rng(21)
    for _ in range(40):
        cnt = int(rng.integers(1, 60))
        m = int(rng.integers(1, 9))
        cost = rng.integers(1, 6, size=cnt).astype(float)
        order = rng.permutation(cnt)
        mach, loads = S.sperm_list_schedule(cost, order, m)
        om, ol = ls(list(cost), list(order), m)
        assert list(mach) == list(om) and np.allclose(loads, ol)
        assert abs(S.replay_efficiency(cost, order, m) - cost.sum() / (m * max(ol))) < 1e-12
    with pytest.raises(S.SpermError):
        S.sperm_list_schedule([1.0, 2.0], [0, 0], 2)


def test_interpolate_mod_matches_exact_lagrange():
    """sperm_interpolate_mod (Newton mod p, host C++) + sperm_crt = exact rational Lagrange
    (oracle.permanent.polynomial_from_values) on random integer polynomials, points spread
    around 0 and arbitrary distinct points."""
    from oracle.permanent import polynomial_from_values
    rng = np.random.default_rng(19)
    for _ in range(25):
        deg = int(rng.integers(0, 30))
        coef = [int(c) for c in rng.integers(-10**12, 10**12, size=deg + 1)]
        xs = list(range(-(deg // 2), deg + 1 - deg // 2)) if rng.random() < 0.5 else \
            [int(v) for v in rng.choice(np.arange(-200, 200), size=deg + 1, replace=False)]
        vals = [sum(c * x ** t for t, c in enumerate(coef)) for x in xs]
        assert polynomial_from_values(xs, vals) == coef
        k = 3
        res = np.array([[v % S.sperm_prime(q) for q in range(S.KMAX)] for v in vals], dtype=np.uint64).astype(np.uint32)
        got = S.residues_to_ints(S.sperm_interpolate_mod(res, xs, k), k)
        assert got == coef
    with pytest.raises(S.SpermError):
        S.sperm_interpolate_mod(np.zeros((2, 8), dtype=np.uint32), [3, 3], 2)
