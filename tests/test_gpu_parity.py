"""GPU parity tests (-m gpu): the CUDA path through the C ABI against the CPU
oracle, element by element, on seeded inputs.  Exact (bit-for-bit) for every
permanent, job list and schedule; KKLLL estimates bit-identical (the 1e-12
relative tolerance of north_star is asserted as the bar)."""
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1112_6072_b200 as P  # noqa: E402
from paper_1112_6072_b200 import pipeline  # noqa: E402
from oracle.cryser import per_ryser_nw_c  # noqa: E402
from oracle.hybrid import expand_to_leaves, h_per, node_permanent, pre_expand, to_dense, to_rows  # noqa: E402
from oracle.kklll import kklll_estimate, kklll_trial  # noqa: E402
from oracle.permanent import per_bruteforce, per_ryser_nw_gray  # noqa: E402
from workloads import dodecahedron, random_3perm, random_3perm_batch, truncated_icosahedron  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    for ln in open(os.path.join(GOLD, "oracle_values.txt")):
        if ln.startswith(name + " "):
            return int(ln.split()[1])
    raise KeyError(name)


def dev(x, dtype=torch.int32):
    return torch.tensor(np.asarray(x), dtype=dtype, device="cuda")


def gpu_per(mats, coef=None, min_primes=1, order=None):
    res, k = P.sperm_permanent(dev(mats), coef=None if coef is None else dev(coef, torch.int64),
                               min_primes=min_primes, order=None if order is None else dev(order))
    return P.residues_to_ints(res, k)


# ------------------------------------------------------------------ R-NW
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 13, 16, 17])
def test_rnw_random_signed_small(n):
    rng = np.random.default_rng(100 + n)
    cnt = 37  # ragged batch
    mats = (rng.integers(-4, 6, size=(cnt, n, n)) * (rng.random((cnt, n, n)) < 0.5)).astype(np.int64)
    mats[0] = 0
    if n > 1:
        mats[1, n // 2] = 0  # zero row
    got = gpu_per(mats)
    want = [per_ryser_nw_gray(m) if n <= 13 else h_per(m) for m in mats]
    assert got == want


def test_rnw_config2_full_batch():
    """configs[1]: 256 seeded n=24 3-regular matrices, half 0/1, half weighted in [1,7]."""
    mats = random_3perm_batch(256, 24, seed=2024)
    got = gpu_per(mats)
    want = [h_per(m) for m in mats]
    assert got == want
    for i in (0, 200):  # and the oracle's own R-NW on samples
        assert got[i] == per_ryser_nw_c(mats[i])


def test_rnw_closed_forms_large_orders():
    """per(J_n) = n!, per(J_n - I_n) = D_n at orders spanning every register tile size."""
    D = [1, 0]
    for k in range(2, 41):
        D.append((k - 1) * (D[-1] + D[-2]))
    for n in (10, 20, 23, 24, 25, 31, 32, 33):
        J = np.ones((1, n, n), dtype=np.int64)
        assert gpu_per(J) == [math.factorial(n)]
        assert gpu_per(J - np.eye(n, dtype=np.int64)) == [D[n]]


def test_rnw_block_diagonal_n40():
    """n = 40 (the NP = 40 tile): per of a block-diagonal matrix = product of the blocks'."""
    rng = np.random.default_rng(40)
    blocks = [rng.integers(-3, 4, size=(8, 8)) for _ in range(5)]
    a = np.zeros((40, 40), dtype=np.int64)
    for b, blk in enumerate(blocks):
        a[8 * b:8 * b + 8, 8 * b:8 * b + 8] = blk
    p = rng.permutation(40)
    want = math.prod(per_bruteforce(b) for b in blocks)
    assert gpu_per(a[p][:, rng.permutation(40)][None]) == [want]


def test_rnw_edge_cases():
    # empty batch
    res, k = P.sperm_permanent(torch.zeros((0, 5, 5), dtype=torch.int32, device="cuda"))
    assert res.shape == (0, P.KMAX)
    # order 0: per of the empty matrix is 1 (times coef)
    assert gpu_per(np.zeros((2, 0, 0)), coef=[1, -3]) == [1, -3]
    # huge entries: many primes and small groups (k up to 8)
    rng = np.random.default_rng(8)
    a = rng.integers(-2**21, 2**21, size=(3, 10, 10))
    assert gpu_per(a) == [h_per(m) for m in a]
    # coefficients and min_primes
    mats = random_3perm_batch(5, 11, seed=3)
    cf = [1, -2, 7, 10**12, -(10**15)]
    assert gpu_per(mats, coef=cf, min_primes=4) == [c * per_ryser_nw_c(m) for c, m in zip(cf, mats)]
    # row abs sum >= 2^30 is refused, not wrapped
    with pytest.raises(P.SpermError):
        gpu_per(np.full((1, 4, 4), 2**28))


def test_rnw_order_and_job_accumulators():
    mats = random_3perm_batch(40, 14, seed=9)
    want = [per_ryser_nw_c(m) for m in mats]
    order = np.random.default_rng(1).permutation(40)
    assert gpu_per(mats, order=order) == want
    job = np.arange(40) % 7
    acc = torch.zeros((8, P.KMAX), dtype=torch.int64, device="cuda")
    P.sperm_permanent(dev(mats), job=dev(job), num_jobs=7, min_primes=2, job_acc=acc)
    red = P.sperm_reduce_mod(acc).cpu().numpy().view(np.uint32)
    for j in range(7):
        assert P.sperm_crt(red[j], 2) == sum(w for w, jj in zip(want, job) if jj == j)
    assert P.sperm_crt(red[7], 2) == sum(want)


def test_rnw_lifted_one_prime_leaves():
    """Leaves whose |coef| * bound fits one (two) primes are evaluated mod p_0 (p_1) and lifted to min_primes
    residues in the finalize: every residue (signed values, signed coefficients, zero, mixed with
    leaves that need several primes) equals the exact value mod p_q, and equals the unlifted run
    (SPERM_LIFT=0)."""
    rng = np.random.default_rng(31)
    mats = rng.integers(-3, 4, size=(48, 12, 12)) * (rng.random((48, 12, 12)) < 0.35)
    mats[5] = 0
    mats[7] = rng.integers(-2**8, 2**8, size=(12, 12))  # needs several primes itself
    mats[11] = rng.integers(-4, 5, size=(12, 12))  # two primes: lifted by Garner's step
    cf = rng.integers(-9, 10, size=48)
    cf[9] = 10**12
    want = [int(c) * h_per(m) for c, m in zip(cf, mats)]
    runs = []
    for lift in ("1", "0"):
        os.environ["SPERM_LIFT"] = lift
        try:
            res, k = P.sperm_permanent(dev(mats), coef=dev(cf, torch.int64), min_primes=4)
        finally:
            os.environ.pop("SPERM_LIFT", None)
        r = res.cpu().numpy().view(np.uint32)
        kk = k.cpu().numpy()
        assert (kk >= 4).all()
        for i, w in enumerate(want):
            for q in range(kk[i]):
                assert int(r[i, q]) == w % P.sperm_prime(q), (lift, i, q)
        assert P.residues_to_ints(res, k) == want
        runs.append(r.copy())
    assert (runs[0] == runs[1]).all()


# ------------------------------------------------------------------ expansion
def _gpu_jobs(a, J):
    sets = pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=J)
    out = []
    for s in sets:
        m, c = s.mats.cpu().numpy(), s.coef.cpu().numpy()
        for i in range(s.count):
            out.append((int(c[i]), m[i].tolist()))
    return out


def _oracle_jobs(a, J):
    return [(c, to_dense(m, k)) for c, m, k in pre_expand(a, jobs_at_least=J)]


def test_expand_c20_identical_job_lists():
    a = dodecahedron()
    for J in (1, 2, 5, 17, 64, 200):
        assert _gpu_jobs(a, J) == _oracle_jobs(a, J)


def test_expand_c60_many_tiles_identical():
    """Levels of thousands of nodes: the single-pass look-back spans hundreds of 8-node tiles
    (beyond its 32-tile window), and the job list still equals the oracle's, in order."""
    a = truncated_icosahedron()
    assert _gpu_jobs(a, 3000) == _oracle_jobs(a, 3000)


def test_expand_capacity_and_null_outputs():
    """Raw C ABI: too small an output capacity -> SPERM_ERR_CAPACITY with the needed counts;
    NULL output buffers with children to write -> SPERM_ERR_ARG."""
    import ctypes
    a = truncated_icosahedron()
    s = pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=500)[0]
    (km, _, _), (em, _, _) = P.sperm_expand(s.mats, s.coef, s.job)
    need = km.shape[0]
    n = s.n
    L = P.sperm.lib()
    oc, ec = ctypes.c_int64(0), ctypes.c_int64(0)
    small = need // 2
    om = torch.empty((max(small, 1), n - 1, n - 1), dtype=torch.int32, device="cuda")
    ocf = torch.empty(max(small, 1), dtype=torch.int64, device="cuda")
    oj = torch.empty(max(small, 1), dtype=torch.int32, device="cuda")
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    rc = L.sperm_expand(ptr(s.mats), ptr(s.coef), ptr(s.job), n, s.count, ptr(om), ptr(ocf), ptr(oj), small,
                        None, None, None, 0, ctypes.byref(oc), ctypes.byref(ec), None)
    assert rc == P.sperm.ERR_CAPACITY and oc.value == need and ec.value == em.shape[0]
    rc = L.sperm_expand(ptr(s.mats), ptr(s.coef), ptr(s.job), n, s.count, None, None, None, 2 * s.count,
                        None, None, None, s.count, ctypes.byref(oc), ctypes.byref(ec), None)
    assert rc == P.sperm.ERR_ARG and oc.value == need
    torch.cuda.synchronize()


def test_expand_random_signed_identical():
    """Row and column pivots, s = 1..4, zero-line children, s >= 5 early nodes."""
    rng = np.random.default_rng(77)
    for t in range(60):
        n = int(rng.integers(3, 13))
        dens = float(rng.uniform(0.2, 0.8))
        a = (rng.integers(-3, 5, size=(n, n)) * (rng.random((n, n)) < dens)).astype(np.int64)
        a += np.diag(rng.integers(1, 3, size=n))
        J = int(rng.integers(1, 40))
        assert _gpu_jobs(a, J) == _oracle_jobs(a, J), t


def test_expand_conserves_permanent():
    a = truncated_icosahedron()
    sets = pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=64)
    tot = 0
    for s in sets:
        for lv in pipeline.expand_to_leaves(s, 22):
            res, k = P.sperm_permanent(lv.mats, coef=lv.coef, min_primes=2)
            tot += sum(P.residues_to_ints(res, k))
    assert tot == golden("C60_truncated_icosahedron")


def _leaf_multiset(mats, coef, job):
    m = mats.cpu().numpy()
    c = coef.cpu().numpy()
    j = job.cpu().numpy()
    return sorted((int(j[i]), int(c[i]), m[i].tobytes()) for i in range(m.shape[0]))


def _oracle_leaf_multiset(roots, L, pad_to):
    """oracle.expand_to_leaves of every root (dense numpy [count, n, n], coefs, job ids): the
    order-L leaves, and the s >= 5 nodes padded to order pad_to by an identity block."""
    leaves, early = [], []
    for a, c, j in roots:
        rows, n = to_rows(a)
        for cf, m, k in expand_to_leaves((int(c), rows, n), L):
            d = np.array(to_dense(m, k), dtype=np.int32)
            if k == L:
                leaves.append((int(j), int(cf), d.tobytes()))
            else:
                e = np.eye(pad_to, dtype=np.int32)
                e[:k, :k] = d
                early.append((int(j), int(cf), e.tobytes()))
    return sorted(leaves), sorted(early)


@pytest.mark.parametrize("L", [14, 20, 24])
def test_subtree_leaves_equal_oracle_c60(L):
    """sperm_expand_subtree (depth first, in shared memory): the leaves of C60 nodes of order
    L + 4..8 are the same multiset (job, coefficient, every entry) as the oracle's H_per
    recursion (expand_to_leaves) produces from the same nodes."""
    a = truncated_icosahedron()
    n0 = min(32, L + (8 if L < 20 else 4))
    s = pipeline.expand_to_leaves(pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=64)[0], n0)[0]
    assert s.n == n0
    take = min(s.count, 120 if L < 20 else 40)
    roots = [(s.mats[i].cpu().numpy(), int(s.coef[i]), int(s.job[i])) for i in range(take)]
    r = P.sperm_expand_subtree(s.mats[:take], L, 1 << 20, s.coef[:take], s.job[:take])
    (lm, lc, lj), (em, ec, ej) = r
    want_leaves, want_early = _oracle_leaf_multiset(roots, L, n0)
    assert _leaf_multiset(lm, lc, lj) == want_leaves
    assert _leaf_multiset(em, ec, ej) == want_early == []


def test_subtree_random_signed_with_early_nodes():
    """Signed random matrices of order 12-16 (row and column pivots, s = 1..4 merges and minors,
    zero-line children, s >= 5 nodes): leaves and identity-padded early nodes equal the
    oracle's; a too small leaf capacity reports None (re-run on fewer nodes)."""
    rng = np.random.default_rng(91)
    for t in range(12):
        n = int(rng.integers(12, 17))
        dens = float(rng.uniform(0.15, 0.45))
        cnt = 6
        mats = (rng.integers(-3, 5, size=(cnt, n, n)) * (rng.random((cnt, n, n)) < dens)).astype(np.int32)
        mats += np.eye(n, dtype=np.int32)[None] * rng.integers(1, 3, size=(cnt, 1, 1)).astype(np.int32)
        coef = rng.integers(-5, 6, size=cnt)
        L = int(rng.integers(max(2, n - 8), n))
        job = np.arange(cnt, dtype=np.int32) * 3 + 1
        r = P.sperm_expand_subtree(dev(mats), L, 1 << 16, dev(coef, torch.int64), dev(job))
        (lm, lc, lj), (em, ec, ej) = r
        want_leaves, want_early = _oracle_leaf_multiset(list(zip(mats, coef, job)), L, n)
        assert _leaf_multiset(lm, lc, lj) == want_leaves, t
        assert _leaf_multiset(em, ec, ej) == want_early, t
        if len(want_leaves) > 1:
            assert P.sperm_expand_subtree(dev(mats), L, len(want_leaves) - 1, dev(coef, torch.int64), dev(job)) is None


def test_subtree_argument_errors():
    """n > 32, L >= n and NULL outputs are SPERM_ERR_ARG; an empty batch returns nothing."""
    import ctypes
    L = P.sperm.lib()
    oc, ec = ctypes.c_int64(0), ctypes.c_int64(0)
    m = torch.zeros((2, 33, 33), dtype=torch.int32, device="cuda")
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    assert L.sperm_expand_subtree(ptr(m), None, None, 33, 2, 20, None, None, None, 0, None, None, None, 0,
                                  ctypes.byref(oc), ctypes.byref(ec), None) == P.sperm.ERR_ARG
    m = torch.eye(20, dtype=torch.int32, device="cuda")[None].repeat(2, 1, 1)
    assert L.sperm_expand_subtree(ptr(m), None, None, 20, 2, 20, None, None, None, 0, None, None, None, 0,
                                  ctypes.byref(oc), ctypes.byref(ec), None) == P.sperm.ERR_ARG
    assert L.sperm_expand_subtree(ptr(m), None, None, 20, 2, 10, None, None, None, 8, None, None, None, 0,
                                  ctypes.byref(oc), ctypes.byref(ec), None) == P.sperm.ERR_ARG
    (lm, _, _), (em, _, _) = P.sperm_expand_subtree(m[:0], 10, 4)
    assert lm.shape == (0, 10, 10) and em.shape[0] == 0
    # identity: every node is s = 1 down to the leaf, one leaf per root, coefficient 1
    (lm, lc, lj), _ = P.sperm_expand_subtree(m, 10, 4)
    assert lm.shape[0] == 2 and (lm.cpu() == torch.eye(10, dtype=torch.int32)).all() and lc.tolist() == [1, 1]


# ------------------------------------------------------------------ KKLLL
def test_kklll_bit_exact_trials():
    rng = np.random.default_rng(5)
    for n in (1, 2, 3, 5, 8, 13, 24):
        mats = (rng.random((3, n, n)) < 0.4).astype(np.int64)
        mats[:, np.arange(n), np.arange(n)] = 1
        est, xs = P.sperm_estimate(dev(mats), trials=25, seed=11, keep_trials=True)
        xs = xs.cpu().numpy()
        for j in range(3):
            ref = [kklll_trial(mats[j], 11, j, t) for t in range(25)]
            assert np.array_equal(xs[j], np.array(ref)), (n, j)
            e = kklll_estimate(mats[j], 25, 11, j)
            assert abs(float(est[j]) - e) <= 1e-12 * abs(e)


@pytest.mark.parametrize("n", [25, 26, 27, 28, 29, 30, 31, 32, 33, 36, 39, 47, 64, 65, 77, 96, 100, 112])
def test_kklll_bit_exact_large_orders(n):
    """Warp-per-trial kernel (n <= 32) and shared-memory kernel with 64 (n < 40; n >= 34 has more trailing columns than update
    threads), 128 (n < 48) and 256 threads (SPERM_KKLLL_T64_MAX / _T128_MAX move the bounds):
    every trial bit-identical to the oracle, including singular (zero) trials (24 trials:
    ~1e4-1e5 multiplier quotients per order through the reciprocal-based division)."""
    rng = np.random.default_rng(n)
    mats = (rng.random((2, n, n)) < 3.5 / n).astype(np.int64)
    mats[:, np.arange(n), np.arange(n)] = 1
    mats[1, :, 0] = 0  # a zero column: |det| = 0 in every trial
    est, xs = P.sperm_estimate(dev(mats), trials=24, seed=3, keep_trials=True)
    xs = xs.cpu().numpy()
    for j in range(2):
        ref = [kklll_trial(mats[j], 3, j, t) for t in range(24)]
        assert np.array_equal(xs[j], np.array(ref)), (n, j)
    assert (xs[1] == 0).all()


def test_kklll_warp_kernel_every_order(monkeypatch):
    """The warp-per-trial kernel on every order 1..32 (its default range; SPERM_KKLLL_WARP_MIN=1
    pins it): every trial bit-identical to the oracle — sparse job-like patterns,
    a denser pattern (many rows per elimination step: several passes of the 4-row update), a zero
    column (singular in every trial) and C60 job matrices of order 32 with their job ids."""
    monkeypatch.setenv("SPERM_KKLLL_WARP_MIN", "1")
    for n in list(range(1, 33)):
        rng = np.random.default_rng(100 + n)
        mats = (rng.random((3, n, n)) < min(1.0, 3.5 / n)).astype(np.int64)
        mats[2] = (rng.random((n, n)) < 0.6).astype(np.int64)
        mats[:, np.arange(n), np.arange(n)] = 1
        if n > 1:
            mats[1, :, n // 2] = 0
        T = 6 if n > 8 else 12
        est, xs = P.sperm_estimate(dev(mats), trials=T, seed=21, keep_trials=True)
        xs = xs.cpu().numpy()
        for j in range(3):
            ref = [kklll_trial(mats[j], 21, j, t) for t in range(T)]
            assert np.array_equal(xs[j], np.array(ref)), (n, j)
        if n > 1:
            assert (xs[1] == 0).all()
    jobs = pre_expand(truncated_icosahedron(), jobs_at_least=992)
    mats = np.array([to_dense(m, k) for _, m, k in jobs[:3]], dtype=np.int64)
    assert mats.shape[1] == 32
    ids = [7, 1000, 3]
    est, xs = P.sperm_estimate(dev(mats), trials=5, seed=9, keep_trials=True, ids=dev(ids))
    xs = xs.cpu().numpy()
    for j in range(3):
        assert np.array_equal(xs[j], np.array([kklll_trial(mats[j], 9, ids[j], t) for t in range(5)])), j


def test_kklll_cta_kernel_small_orders(monkeypatch):
    """SPERM_KKLLL_WARP_MIN=33 (the A-B knob) sends orders <= 32 to the CTA shared-memory kernel
    instead of the warp kernel: the same bit-identical trials."""
    monkeypatch.setenv("SPERM_KKLLL_WARP_MIN", "33")
    for n in (2, 5, 16, 24, 30, 32):
        rng = np.random.default_rng(300 + n)
        mats = (rng.random((2, n, n)) < min(1.0, 3.5 / n)).astype(np.int64)
        mats[:, np.arange(n), np.arange(n)] = 1
        est, xs = P.sperm_estimate(dev(mats), trials=6, seed=4, keep_trials=True)
        xs = xs.cpu().numpy()
        for j in range(2):
            assert np.array_equal(xs[j], np.array([kklll_trial(mats[j], 4, j, t) for t in range(6)])), (n, j)


def test_kklll_frontal_bit_exact_on_job_matrices():
    """The frontal warp-per-trial kernel (orders >= 48) on whole-path job matrices (C60 jobs of
    order 48, fullerene n=70 jobs of order 51): every trial bit-identical to the oracle, and the
    frontal path (not the CTA fallback) handled the jobs; a dense matrix overflows the front and is
    re-run by the CTA kernel, still exact."""
    from workloads import random_fullerene
    P.sperm_estimate_stats(reset=True)
    for a, J, take, T in ((truncated_icosahedron(), 16, 3, 8), (random_fullerene(70, 2024, 1)[0], 80, 2, 6)):
        jobs = pre_expand(a, jobs_at_least=J)
        mats = np.array([to_dense(m, k) for _, m, k in jobs[:take]], dtype=np.int64)
        assert mats.shape[1] >= 48
        est, xs = P.sperm_estimate(dev(mats), trials=T, seed=9, keep_trials=True)
        xs = xs.cpu().numpy()
        for j in range(take):
            ref = [kklll_trial(mats[j], 9, j, t) for t in range(T)]
            assert np.array_equal(xs[j], np.array(ref)), j
    jobs_front, redo = P.sperm_estimate_stats(reset=True)
    assert jobs_front == 5 and redo == 0
    rng = np.random.default_rng(2)
    dense = (rng.random((1, 50, 50)) < 0.5).astype(np.int64)
    est, xs = P.sperm_estimate(dev(dense), trials=4, seed=1, keep_trials=True)
    assert np.array_equal(xs.cpu().numpy()[0], np.array([kklll_trial(dense[0], 1, 0, t) for t in range(4)]))
    assert P.sperm_estimate_stats(reset=True) == (1.0, 1.0)


def test_kklll_ids_and_default_trials():
    a = dodecahedron()
    est = P.sperm_estimate(dev(a[None]), trials=0, seed=3, ids=dev([5]))
    assert abs(float(est[0]) - kklll_estimate(a, 0, 3, 5)) <= 1e-12 * float(est[0])


# ------------------------------------------------------------------ whole path
@pytest.mark.parametrize("policy", ["estimate", "natural", "random"])
def test_pipeline_c20(policy):
    a = dodecahedron()
    for J, L in ((1, 20), (8, 12), (30, 8), (200, 4)):
        r = pipeline.permanent(a, jobs_at_least=J, leaf_order=L, policy=policy)
        assert r.value == golden("C20_dodecahedron")
        oj = pre_expand(a, jobs_at_least=J)
        assert r.job_values == [node_permanent(j) for j in oj]


def test_pipeline_random_sparse_vs_hper():
    rng = np.random.default_rng(31)
    for _ in range(12):
        n = int(rng.integers(8, 19))
        a = (rng.random((n, n)) < 0.25).astype(np.int64) * rng.integers(1, 4, size=(n, n))
        a += np.eye(n, dtype=np.int64)
        r = pipeline.permanent(a, jobs_at_least=int(rng.integers(1, 30)), leaf_order=int(rng.integers(3, 12)))
        assert r.value == h_per(a)


def test_pipeline_fullerenes_config4():
    """configs[3]: seeded spiral fullerenes n in {70,76,80,84}, 4 isomers each, exact per(A)
    against the oracle's frontier-DP values (tests/golden/oracle_values.txt)."""
    from workloads import random_fullerene
    checked = 0
    for n in (70, 76, 80, 84):
        for iso in range(4):
            try:
                want = golden(f"fullerene_n{n}_seed2024_iso{iso}")
            except KeyError:
                continue
            a, _ = random_fullerene(n, 2024, iso)
            r = pipeline.permanent(a, jobs_at_least=256, leaf_order=22)
            assert r.value == want, (n, iso)
            checked += 1
    assert checked >= 12


def test_pipeline_streamed_leaves_tiny_budget():
    """iter_leaves splits levels that would exceed the HBM budget into chunks (depth first):
    a 256 KB budget forces many splits; per-job values and the total must not change."""
    a = truncated_icosahedron()
    r1 = pipeline.permanent(a, jobs_at_least=16, leaf_order=24)
    r2 = pipeline.permanent(a, jobs_at_least=16, leaf_order=24, leaf_budget_bytes=256 << 10)
    assert r1.value == r2.value == golden("C60_truncated_icosahedron")
    assert r1.job_values == r2.job_values and r1.leaves == r2.leaves


def test_pipeline_measure_jobs_and_signed_input():
    """Per-job cycle counters are filled for every job; a signed matrix (no prime cap)."""
    a = dodecahedron()
    r = pipeline.permanent(a, jobs_at_least=12, leaf_order=10, measure_jobs=True)
    assert r.value == 1392 and len(r.job_cycles) == r.num_jobs and (r.job_cycles > 0).all()
    rng = np.random.default_rng(4)
    b = a * rng.choice([-3, -1, 2, 5], size=a.shape)
    assert pipeline.permanent(b, jobs_at_least=20, leaf_order=12).value == h_per(b)


def test_pipeline_dynamic_assignment_single_rank():
    """assignment="dynamic" with an explicit store (one rank): chunks claimed from the store's
    counter map back to their job sets; value and every job value unchanged."""
    import socket
    from torch.distributed import TCPStore
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    store = TCPStore("127.0.0.1", port, 1, True)
    a = truncated_icosahedron()
    r1 = pipeline.permanent(a, jobs_at_least=128, leaf_order=18)
    r2 = pipeline.permanent(a, jobs_at_least=128, leaf_order=18, assignment="dynamic", store=store, dynamic_chunk=5)
    assert r2.value == r1.value == golden("C60_truncated_icosahedron")
    assert r2.job_values == r1.job_values
    assert r2.stats["claims"] == -(-r1.num_jobs // 5) + 1  # device queue: every chunk + the empty claim
    r3 = pipeline.permanent(a, jobs_at_least=128, leaf_order=18, assignment="dynamic", store=store, dynamic_chunk=7,
                            queue="store")
    assert r3.job_values == r1.job_values


def test_pipeline_c60_l32_every_job():
    """configs[2] as the bench runs it: C60, J >= 992 jobs, leaves of order <= 32 — every one of
    the job values equals the oracle's (Python pre-expansion, per job by the C frontier DP)."""
    from oracle.cfrontier import narrow_order, per_frontier_c
    a = truncated_icosahedron()
    r = pipeline.permanent(a, jobs_at_least=992, leaf_order=32)
    assert r.value == golden("C60_truncated_icosahedron")
    jobs = pre_expand(a, jobs_at_least=992)
    assert r.num_jobs == len(jobs)
    want = []
    for c, m, k in jobs:
        d = np.array(to_dense(m, k), dtype=np.int64)
        want.append(c * per_frontier_c(d, narrow_order(d)))
    assert r.job_values == want


def test_pipeline_fold_every_leaf_set():
    """The uint64 accumulators folded mod p (sperm_fold_mod) before every leaf set: the same
    per-job values and total as without folding."""
    a = truncated_icosahedron()
    r1 = pipeline.permanent(a, jobs_at_least=128, leaf_order=20)
    r2 = pipeline.permanent(a, jobs_at_least=128, leaf_order=20, fold_every=1, leaf_budget_bytes=256 << 10)
    assert r2.stats.get("folds", 0) >= 2
    assert r1.value == r2.value == golden("C60_truncated_icosahedron")
    assert r1.job_values == r2.job_values
    acc = torch.tensor([[2**63 + 5] * 8, [123] * 8], dtype=torch.uint64).view(torch.int64).cuda()
    P.sperm_fold_mod(acc)
    got = acc.cpu().view(torch.uint64).numpy().astype(object)
    for q in range(P.KMAX):
        assert int(got[0, q]) == (2**63 + 5) % P.sperm_prime(q) and int(got[1, q]) == 123


def test_pipeline_c60_leaf16():
    a = truncated_icosahedron()
    r = pipeline.permanent(a, jobs_at_least=128, leaf_order=18)
    assert r.value == golden("C60_truncated_icosahedron")


# ------------------------------------------------------------------ R-NW kernel variants
def _plans_agree(mats, want):
    """Every tree plan (forced via SPERM_RNW_PLAN_MIN) and the generic kernel agree with the oracle."""
    for pmin in ("1", "2", "3", "4", "5", "0"):
        os.environ["SPERM_RNW_PLAN_MIN"] = pmin
        try:
            got = gpu_per(mats)
        finally:
            os.environ.pop("SPERM_RNW_PLAN_MIN", None)
        assert got == want, pmin


def test_rnw_speculative_groups_repeat_and_change():
    """Same-shape calls launch the previous call's plan groups before the histogram read-back
    (csrc/rnw.cu rnw_spec_check_kernel): repeats, same-shape batches with other contents and other
    plan histograms must all stay exact (SPERM_SPECULATE=1 forces it on)."""
    os.environ["SPERM_SPECULATE"] = "1"
    try:
        _speculative_cases()
    finally:
        os.environ.pop("SPERM_SPECULATE", None)


def _speculative_cases():
    a = random_3perm_batch(16, 20, seed=11)
    a2 = random_3perm_batch(16, 20, seed=12)
    rng = np.random.default_rng(7)
    b = (rng.integers(-3, 4, size=(16, 20, 20)) * (rng.random((16, 20, 20)) < 0.2)).astype(np.int64)
    want = {id(x): [h_per(m) for m in x] for x in (a, a2, b)}
    want_a = want[id(a)]
    for x in (a, a, a2, b, b, a, a2, a2):
        assert gpu_per(x) == want[id(x)]
    # above the single-CTA grouping size (keys kernel + radix sort + separate check kernel)
    c = random_3perm_batch(5000, 12, seed=13)
    c2 = c.copy()
    c2[::3] = (rng.integers(-3, 4, size=(1667, 12, 12)) * (rng.random((1667, 12, 12)) < 0.4)).astype(np.int64)
    want = {id(x): [per_ryser_nw_c(m) for m in x] for x in (c, c2)}
    for x in (c, c, c2, c2, c):
        assert gpu_per(x) == want[id(x)]
    # a same-shape call whose prep reports an error: the speculative groups must not run, the
    # error is raised, and the next call is exact again
    bad = a.copy()
    bad[3, 5, :] = 1 << 26  # row abs sum 20 * 2^26 >= 2^30
    gpu_per(a)
    with pytest.raises(P.SpermError):
        gpu_per(bad)
    assert gpu_per(a) == want_a


def test_rnw_tree_plans_3regular():
    for n, seed in ((12, 1), (17, 2), (20, 3), (26, 4)):
        mats = random_3perm_batch(12, n, seed=seed)
        _plans_agree(mats, [h_per(m) for m in mats])


def test_rnw_tree_plans_fullerene_leaves():
    """Leaves of the C60 expansion (merged entries, uneven row/column counts)."""
    a = truncated_icosahedron()
    sets = pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=8)
    lv = pipeline.expand_to_leaves(sets[0], 24)[0]
    idx = torch.arange(0, lv.count, max(1, lv.count // 16), device="cuda")[:16]
    mats = lv.mats.index_select(0, idx).cpu().numpy()
    _plans_agree(mats, [h_per(m) for m in mats])


def test_rnw_tree_plans_signed_sparse():
    rng = np.random.default_rng(12)
    mats = []
    for _ in range(10):
        n = int(rng.integers(14, 23))
        a = random_3perm(n, rng) * rng.integers(-5, 6, size=(n, n))
        a[np.arange(n), np.arange(n)] += rng.integers(1, 3, size=n)
        mats.append(a)
    for a in mats:
        _plans_agree(a[None], [h_per(a)])


@pytest.mark.parametrize("wmax", [60, 2000])
def test_rnw_many_primes_every_plan(wmax):
    """Heavy weights need k = 4..8 primes: the tree kernel's generic-K block loop (k > 3) and the
    generic kernel, with every tree plan forced in turn, against the oracle."""
    rng = np.random.default_rng(wmax)
    mats = []
    for _ in range(6):
        n = int(rng.integers(16, 23))
        a = random_3perm(n, rng) * rng.integers(1, wmax + 1, size=(n, n))
        mats.append(a)
    for a in mats:
        res, k = P.sperm_permanent(dev(a[None]))
        assert int(k[0]) >= 4
        _plans_agree(a[None], [h_per(a)])


def _forced(mats, plan_min):
    os.environ["SPERM_RNW_PLAN_MIN"] = plan_min
    try:
        return gpu_per(mats)
    finally:
        os.environ.pop("SPERM_RNW_PLAN_MIN", None)


@pytest.mark.parametrize("n", [27, 30, 33, 36, 40])
def test_rnw_per_leaf_orders_27_to_40_every_fixed_width(n):
    """Leaves of orders 27-40, one by one against the C frontier DP.  With a plan forced to few
    low columns (SPERM_RNW_PLAN_MIN: plan 8 = B 1, plan 12 = B 2 with pairs; plan 6 = B 3) the
    fixed rows n - 3B select the wide fixed-row tables: NFIX 24 (n - 3B <= 24), 32 and 40;
    the default plan (B = 8) covers NFIX 4-16.  Signed weights on two of the leaves."""
    from oracle.cfrontier import narrow_order, per_frontier_c
    rng = np.random.default_rng(1000 + n)
    mats = [random_3perm(n, rng) for _ in range(3)]
    mats[1] = mats[1] * rng.integers(1, 4, size=(n, n))
    mats[2] = mats[2] * rng.choice([-2, -1, 1, 3], size=(n, n))
    mats = np.array(mats)
    want = [per_frontier_c(m, narrow_order(m)) for m in mats]
    assert gpu_per(mats) == want
    for plan_min in ("6", "8", "12"):
        assert _forced(mats, plan_min) == want, plan_min
    if n <= 30:
        assert _forced(mats, "0") == want  # the generic kernel


def test_rnw_per_leaf_c60_l32_leaves():
    """Order-32 leaves of configs[2] (C60 expanded to J >= 992 jobs; merged entries), one by one
    against the frontier DP, under the default plan and forced narrow plans."""
    from oracle.cfrontier import narrow_order, per_frontier_c
    a = truncated_icosahedron()
    sets = pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=992)
    s = [x for x in sets if x.n == 32][0]
    idx = torch.arange(0, s.count, max(1, s.count // 12), device="cuda")[:12]
    mats = s.mats.index_select(0, idx).cpu().numpy().astype(np.int64)
    want = [per_frontier_c(m, narrow_order(m)) for m in mats]
    assert gpu_per(mats) == want
    for plan_min in ("4", "8", "12"):
        assert _forced(mats, plan_min) == want, plan_min


@pytest.mark.parametrize("n", [44, 48])
def test_rnw_per_leaf_max_orders(n):
    """The largest leaves (SPERM_NMAX = 48: 2^47 Gray-code terms), one 3-regular and one
    weighted, against the frontier DP."""
    from oracle.cfrontier import narrow_order, per_frontier_c
    rng = np.random.default_rng(2000 + n)
    mats = np.array([random_3perm(n, rng), random_3perm(n, rng) * rng.integers(1, 3, size=(n, n))])
    want = [per_frontier_c(m, narrow_order(m)) for m in mats]
    assert gpu_per(mats) == want


def test_crt_device_matches_host():
    """sperm_crt_device (GPU Garner + limbs) = sperm_crt (host) on random residues, every k, signs."""
    rng = np.random.default_rng(9)
    res = rng.integers(0, 2**31 - 1, size=(300, P.KMAX), dtype=np.int64).astype(np.uint32)
    ks = rng.integers(1, P.KMAX + 1, size=300).astype(np.int32)
    res[0, :] = 0  # zero
    got = P.residues_to_ints_device(torch.tensor(res.view(np.int32), device="cuda"),
                                    torch.tensor(ks, device="cuda"))
    want = [P.sperm_crt(res[i], int(ks[i])) for i in range(300)]
    assert got == want and got[0] == 0 and any(v < 0 for v in got)


def test_rnw_subkey_sort_large_batch(monkeypatch):
    """SPERM_RNW_SUBKEY=1 (measurement knob): a batch above the small-batch limit is ordered inside
    each plan group by prime class and exact-E mode; residues and prime counts are those of the
    default order, and sampled values equal the oracle's."""
    mats = np.concatenate([random_3perm_batch(2600, 12, seed=41), random_3perm_batch(2600, 12, seed=42)])
    mats[2600:] *= np.random.default_rng(3).integers(1, 60, size=(2600, 12, 12))
    d = dev(mats)
    res0, k0 = P.sperm_permanent(d, min_primes=1)
    monkeypatch.setenv("SPERM_RNW_SUBKEY", "1")
    res1, k1 = P.sperm_permanent(d, min_primes=1)
    assert np.array_equal(k0.cpu().numpy(), k1.cpu().numpy()) and np.array_equal(res0.cpu().numpy(), res1.cpu().numpy())
    assert len(set(k1.cpu().tolist())) > 1  # several prime classes in the batch
    got = P.residues_to_ints(res1, k1)
    for j in (0, 17, 2599, 2600, 4000, 5199):
        assert got[j] == per_ryser_nw_gray(mats[j]), j


def test_rnw_prime_count_bregman_and_cap():
    """0/1 leaves size their prime count by Bregman-Minc (configs[1] 0/1 half: 1 prime);
    max_primes caps it, leaving every residue correct modulo the primes kept."""
    mats = random_3perm_batch(256, 24, seed=2024)[[0, 1, 2, 200, 201]]
    res, k = P.sperm_permanent(dev(mats))
    k = k.cpu().numpy()
    assert list(k[:3]) == [1, 1, 1] and all(x >= 3 for x in k[3:])
    want = [h_per(m) for m in mats]
    assert P.residues_to_ints(res, k) == want
    res2, k2 = P.sperm_permanent(dev(mats), min_primes=1, max_primes=2)
    r2 = res2.cpu().numpy().view(np.uint32)
    assert list(k2.cpu().numpy()) == [1, 1, 1, 2, 2]
    for i, w in enumerate(want):
        for q in range(int(k2[i])):
            assert int(r2[i, q]) == w % P.sperm_prime(q)
    with pytest.raises(P.SpermError):
        P.sperm_permanent(dev(mats), min_primes=3, max_primes=2)


# ------------------------------------------------------------------ multi-rank pipeline
def _ws2_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    sys_path_root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import sys
    if sys_path_root not in sys.path:
        sys.path.insert(0, sys_path_root)
    import paper_1112_6072_b200 as P_  # noqa: F401
    from paper_1112_6072_b200 import pipeline as pl
    from workloads import dodecahedron as dod, truncated_icosahedron as ti
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    res = {}
    for name, a, J, L in (("C20", dod(), 30, 8), ("C60", ti(), 128, 18)):
        for policy, asg, q in (("estimate", "static", "device"), ("estimate", "dynamic", "device"),
                               ("estimate", "dynamic", "store"), ("size", "static", "device"),
                               ("natural", "static", "device"), ("random", "static", "device")):
            r = pl.permanent(a, jobs_at_least=J, leaf_order=L, policy=policy, assignment=asg,
                             group=dist.group.WORLD, dynamic_chunk=3, queue=q)
            res[f"{name}_{policy}_{asg}_{q}"] = (r.value, r.job_values, r.machine.tolist(), r.num_jobs,
                                                 r.stats.get("claims", 0))
    import pickle
    with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


def test_pipeline_two_ranks_gloo_same_device(tmp_path):
    """pipeline.permanent with a world-size-2 process group (two processes on cuda:0, gloo: the
    collectives go through the host, so neither rank's kernels wait on the other's): sharded
    KKLLL estimates + all-reduce, replicated LPT schedule, each rank evaluating only its jobs
    (static) or claiming chunks from the store (dynamic), residue all-reduce + CRT.  Both ranks
    must return the exact per(A) and every job value the single-rank run and the oracle give."""
    import socket
    import torch.multiprocessing as mp
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    mp.start_processes(_ws2_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    import pickle
    rs = [pickle.load(open(tmp_path / f"r{r}.pkl", "rb")) for r in range(2)]
    c20_jobs = [node_permanent(j) for j in pre_expand(dodecahedron(), jobs_at_least=30)]
    single_c60 = pipeline.permanent(truncated_icosahedron(), jobs_at_least=128, leaf_order=18)
    for key in rs[0]:
        v0, jv0, mach0, nj, c0 = rs[0][key]
        v1, jv1, mach1, _, c1 = rs[1][key]
        if "dynamic_device" in key:  # IPC-mapped counter: every chunk claimed once over both ranks
            assert c0 + c1 == -(-nj // 3) + 2, key
        if key.endswith("static_device"):
            key = key[:-len("_device")]
        assert v0 == v1 and jv0 == jv1 and mach0 == mach1, key
        if key.startswith("C20"):
            assert v0 == 1392 and jv0 == c20_jobs, key
        else:
            assert v0 == golden("C60_truncated_icosahedron") and jv0 == single_c60.job_values, key
        if key.endswith("static"):
            assert set(mach0) == {0, 1}, key  # both ranks were dealt jobs


@pytest.mark.parametrize("name", ["fullerene_n96_seed2024_iso0", "random3reg_n96_seed2024_96"])
def test_pipeline_configs4_n96_vs_oracle(name):
    """configs[4]: both n = 96 matrices through the whole path (the bench's strong-scaling
    configuration, J >= 160, L = 16; and J >= 1000) against the C frontier DP's values."""
    import numpy as np_
    from workloads import random_fullerene
    if name.startswith("fullerene"):
        a = random_fullerene(96, 2024, 0)[0]
    else:
        a = random_3perm(96, np_.random.default_rng(np_.random.PCG64([2024, 96])))
    want = golden(name)
    for J in (160, 1000):
        r = pipeline.permanent(a, jobs_at_least=J, leaf_order=16)
        assert r.value == want, J
        assert sum(r.job_values) == want


def test_permanent_host_buffers():
    """sperm_permanent_host (host buffers: H2D, R-NW, device CRT, D2H in one call) on configs[1]'s
    first 16 + last 16 matrices and a signed ragged case, against the oracle."""
    mats = random_3perm_batch(256, 24, seed=2024)
    sel = np.concatenate([mats[:16], mats[-16:]]).astype(np.int32)
    assert P.sperm_permanent_host(np.ascontiguousarray(sel)) == [h_per(m) for m in sel]
    rng = np.random.default_rng(17)
    b = (rng.integers(-5, 6, size=(9, 11, 11)) * (rng.random((9, 11, 11)) < 0.4)).astype(np.int32)
    assert P.sperm_permanent_host(b, min_primes=3) == [per_ryser_nw_gray(m) for m in b]
    assert P.sperm_permanent_host(np.zeros((0, 5, 5), dtype=np.int32)) == []


# ------------------------------------------------------------------ NEXT-3: case study 3 and Eq. (11)
def test_permanental_polynomial_c20_and_small():
    """pipeline.permanental_polynomial (R-NW at n + 1 points in one batched call, modular
    interpolation, CRT) = the oracle's polynomial of C20 (frontier values + exact Lagrange) and
    the brute-force expansion of Eq. (11) on random signed matrices n <= 7."""
    from test_oracle import c20_polynomial
    from oracle.permanent import permanental_polynomial as oracle_poly
    assert pipeline.permanental_polynomial(dodecahedron()) == c20_polynomial()
    rng = np.random.default_rng(23)
    for _ in range(12):
        n = int(rng.integers(1, 8))
        a = rng.integers(-4, 5, size=(n, n)) * (rng.random((n, n)) < 0.6)
        assert pipeline.permanental_polynomial(a) == oracle_poly(a)


def test_case_study3_c60_i_plus_a():
    """Case study 3 (Table 4): per(I + A) of C60 — the 4-regular matrix of the
    permanental-polynomial study — through the whole path, against the C frontier DP."""
    from oracle.cfrontier import per_frontier_c
    from oracle.frontier import bfs_order
    a = truncated_icosahedron() + np.eye(60, dtype=np.int64)
    want = per_frontier_c(a, bfs_order(truncated_icosahedron()))
    r = pipeline.permanent(a, jobs_at_least=123, leaf_order=24)
    assert r.value == want


def test_pipeline_auto_leaf_order():
    """leaf_order="auto" (NEXT-1): L measured on a sample of the jobs; the value and every job
    value are those of a fixed-L run, and the choice is one of the timed candidates."""
    a = truncated_icosahedron()
    r = pipeline.permanent(a, jobs_at_least=128, leaf_order="auto")
    r0 = pipeline.permanent(a, jobs_at_least=128, leaf_order=18)
    assert r.value == golden("C60_truncated_icosahedron") and r.job_values == r0.job_values
    times = r.stats["leaf_order_auto"]
    L = r.stats["leaf_order"]
    assert str(L) in times and times[str(L)] == min(times.values())
