"""Small invocation of every libsperm kernel, for compute-sanitizer runs (one tool per run):

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1112_6072_b200 as P  # noqa: E402
from paper_1112_6072_b200 import pipeline  # noqa: E402
from workloads import dodecahedron, random_3perm_batch, truncated_icosahedron  # noqa: E402


def main():
    rng = np.random.default_rng(1)
    # R-NW: tree plans (3-regular, weighted) and the generic kernel (dense signed), ragged sizes
    for n, cnt in ((14, 5), (20, 7), (24, 3)):
        m = torch.tensor(random_3perm_batch(cnt, n, seed=n), dtype=torch.int32, device="cuda")
        P.sperm_permanent(m, min_primes=2)
    d = torch.tensor(rng.integers(-3, 4, size=(6, 9, 9)), dtype=torch.int32, device="cuda")
    P.sperm_permanent(d)
    # KKLLL: register (n <= 32), CTA (32 < n <= 96) and shared-memory (n > 96) kernels
    for n in (7, 24, 40, 100):
        a = (rng.random((2, n, n)) < 3.0 / n).astype(np.int32)
        a[:, np.arange(n), np.arange(n)] = 1
        P.sperm_estimate(torch.tensor(a, device="cuda"), trials=3, seed=2)
    # expansion + the whole path
    assert pipeline.permanent(dodecahedron(), jobs_at_least=16, leaf_order=10).value == 1392
    r = pipeline.permanent(truncated_icosahedron(), jobs_at_least=32, leaf_order=26)
    torch.cuda.synchronize()
    print("sanitize smoke ok", r.value)


if __name__ == "__main__":
    main()
