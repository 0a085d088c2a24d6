import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1112_6072_b200 as P
from paper_1112_6072_b200 import pipeline
from workloads import truncated_icosahedron, dodecahedron
pipeline.permanent(dodecahedron(), jobs_at_least=8, leaf_order=12)
a = truncated_icosahedron() + np.eye(60, dtype=np.int64)
for J, L in ((123, 24), (123, 20), (123, 18), (1000, 18), (1000, 16)):
    P.sperm_timing_enable(True); P.sperm_timing_reset()
    torch.cuda.synchronize(); t = time.perf_counter()
    try:
        r = pipeline.permanent(a, jobs_at_least=J, leaf_order=L)
        torch.cuda.synchronize()
        st = {s: round(P.sperm_timing_get(s)[0], 1) for s in ("expand", "kklll", "rnw_prep", "rnw", "rnw_finalize")}
        print(J, L, r.value, r.num_jobs, r.leaves, round(time.perf_counter() - t, 2), st, flush=True)
    except Exception as e:
        print(J, L, 'ERR', e, flush=True)
t = time.perf_counter()
for n in (20, 24, 28, 32):
    from workloads import random_3perm
    g = random_3perm(n, np.random.default_rng(n))
    g = ((g + g.T) > 0).astype(np.int64)
    t = time.perf_counter()
    c = pipeline.permanental_polynomial(g)
    print('poly', n, round(time.perf_counter() - t, 3), c[:3], flush=True)
