"""Algorithm KKLLL — test infrastructure only.

Estimator: B_ij = 0 where A_ij = 0, else an independent uniform cube root of
unity w0 = 1, w1 = -1/2 + (sqrt3/2) i, w2 = -1/2 - (sqrt3/2) i
(PAPER.md:198-199, 208-213); X_A = det(B) * conj(det(B)) = |det B|^2
(PAPER.md:214).  Theorem 1: E[X_A] = per(A).  The
estimate of a job is the mean over N trials (N = n^2 by default, "the trials
is about n^2").  Weighted matrices are estimated on their 0/1
pattern.

Readings:
  K1  Random choice: counter-based generator (below); root index
      ((h >> 32) * 3) >> 32 of the 64-bit hash h of (seed, job, trial, i, j).
  K2  det by LU with partial pivoting: pivot = first row (lowest index) with
      the maximal |b_ik|^2 = re*re + im*im over rows i >= k; multiplier
      l = b_ik * conj(b_kk) / |b_kk|^2; update b_ij -= l * b_kj for j > k;
      |det|^2 = prod_k |b_kk|^2 in k order; a zero pivot column gives 0.
      Every real operation is a single IEEE-754 round-to-nearest fp64 op, in
      the order written (no fused multiply-add), so the CUDA estimator can be
      bit-identical.
  K3  The mean is the sum over trials in trial order divided by N.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
SQRT3_2 = 0.8660254037844386  # nearest double to sqrt(3)/2
ROOTS = ((1.0, 0.0), (-0.5, SQRT3_2), (-0.5, -SQRT3_2))


def mix64(z: int) -> int:
    """SplitMix64 finaliser (Steele, Lea, Flood 2014), 64-bit wrap-around."""
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def trial_key(seed: int, job: int, trial: int) -> int:
    h = mix64((seed + 0x9E3779B97F4A7C15 * (job + 1)) & M64)
    return mix64(h ^ ((trial * 0xD1B54A32D192ED03) & M64))


def root_index(key: int, i: int, j: int) -> int:
    h = mix64(key ^ ((i << 32) | j))
    return ((h >> 32) * 3) >> 32


def random_b(pattern, seed: int, job: int, trial: int):
    """Step 1 of KKLLL: the randomised matrix B as (re, im) float64 arrays."""
    a = np.asarray(pattern)
    n = a.shape[0]
    re = np.zeros((n, n), dtype=np.float64)
    im = np.zeros((n, n), dtype=np.float64)
    key = trial_key(seed, job, trial)
    for i in range(n):
        for j in range(n):
            if a[i, j] != 0:
                r = ROOTS[root_index(key, i, j)]
                re[i, j] = r[0]
                im[i, j] = r[1]
    return re, im


def det_abs2(re: np.ndarray, im: np.ndarray) -> float:
    """Step 2 of KKLLL: |det B|^2 by LU with partial pivoting (reading K2).
    numpy is used only for elementwise fp64 ops (each one IEEE-rounded)."""
    re = re.copy()
    im = im.copy()
    n = re.shape[0]
    x = 1.0
    for k in range(n):
        mag = re[k:, k] * re[k:, k] + im[k:, k] * im[k:, k]
        p = k + int(np.argmax(mag))  # first maximal entry
        d = float(mag[p - k])
        if d == 0.0:
            return 0.0
        if p != k:
            re[[k, p]] = re[[p, k]]
            im[[k, p]] = im[[p, k]]
        pr, pi = re[k, k], im[k, k]
        x = x * d
        if k + 1 == n:
            break
        xr = re[k + 1:, k]
        xi = im[k + 1:, k]
        lr = (xr * pr + xi * pi) / d
        li = (xi * pr - xr * pi) / d
        ur = re[k, k + 1:]
        ui = im[k, k + 1:]
        re[k + 1:, k + 1:] = re[k + 1:, k + 1:] - (lr[:, None] * ur[None, :] - li[:, None] * ui[None, :])
        im[k + 1:, k + 1:] = im[k + 1:, k + 1:] - (lr[:, None] * ui[None, :] + li[:, None] * ur[None, :])
    return x


def kklll_trial(pattern, seed: int, job: int, trial: int) -> float:
    re, im = random_b(pattern, seed, job, trial)
    return det_abs2(re, im)


def kklll_estimate(pattern, trials: int = 0, seed: int = 1, job: int = 0) -> float:
    """Mean of `trials` KKLLL trials (0 -> n^2), reading K3."""
    a = (np.asarray(pattern) != 0).astype(np.int64)
    n = a.shape[0]
    if trials <= 0:
        trials = n * n
    s = 0.0
    for t in range(trials):
        s = s + kklll_trial(a, seed, job, t)
    return s / trials


def kklll_all_assignments_mean(pattern) -> float:
    """Exact expectation of X_A over all 3^nnz root assignments (Theorem 1,
    PAPER.md:218-220), for tiny matrices; a pin, not an estimator."""
    from itertools import product
    a = np.asarray(pattern)
    n = a.shape[0]
    nz = [(i, j) for i in range(n) for j in range(n) if a[i, j] != 0]
    tot = 0.0
    cnt = 0
    for choice in product(range(3), repeat=len(nz)):
        re = np.zeros((n, n))
        im = np.zeros((n, n))
        for (i, j), c in zip(nz, choice):
            re[i, j], im[i, j] = ROOTS[c]
        tot += det_abs2(re, im)
        cnt += 1
    return tot / cnt
