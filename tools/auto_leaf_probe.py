"""Probe of leaf_order="auto" (NEXT-1) against hand-picked L on the paper's C100 and configs[4].

    python tools/auto_leaf_probe.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1112_6072_b200 import pipeline  # noqa: E402
from workloads import dodecahedron, paper_graph, random_3perm, random_fullerene  # noqa: E402

pipeline.permanent(dodecahedron(), jobs_at_least=8, leaf_order=12)
cases = [("C100", paper_graph("C100"), 159), ("fullerene96", random_fullerene(96, 2024, 0)[0], 160),
         ("random96", random_3perm(96, np.random.default_rng(np.random.PCG64([2024, 96]))), 160)]
for name, a, J in cases:
    for L in ("auto", 15, 16):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = pipeline.permanent(a, jobs_at_least=J, leaf_order=L)
        torch.cuda.synchronize()
        print(json.dumps({"case": name, "L": L, "chosen": r.stats["leaf_order"], "wall_s": time.perf_counter() - t,
                          "per": str(r.value), "auto": r.stats.get("leaf_order_auto")}), flush=True)
