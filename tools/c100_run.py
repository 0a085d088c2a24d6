"""per(C100) — the paper's case study (§4.1, Tables 5-7, Table T12) on one B200.

    python tools/c100_run.py [--jobs 159] [--leaf 20] [--out gpurun_out/c100.json]

The appendix graph (workloads.paper_graph("C100")) is expanded by Algorithm
PH to >= J jobs, KKLLL-weighted, LPT-ordered, expanded to leaves of order <= L and evaluated
by the batched R-NW kernels; the exact total is compared with Table T12's Total,
per(C100) = 149364113290700 (tests/golden/paper_pins.txt).  The paper needed
118413 s on one Pentium III (Table 5) and 3797 s on 32 of them (Table 6).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=159)
    ap.add_argument("--leaf", type=int, default=20)
    ap.add_argument("--budget-gb", type=float, default=16.0, help="HBM budget of a streamed expansion level")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c100.json"))
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_1112_6072_b200 as P
    from paper_1112_6072_b200 import pipeline
    from workloads import dodecahedron, paper_graph

    pin = None
    for ln in open(os.path.join(ROOT, "tests", "golden", "paper_pins.txt")):
        if ln.startswith("per_C100 "):
            pin = int(ln.split()[1])
    a = paper_graph("C100")
    pipeline.permanent(dodecahedron(), jobs_at_least=8, leaf_order=12)  # warm-up
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    P.sperm_rnw_stats(reset=True)
    P.sperm_expand_stats(reset=True)
    t0 = time.perf_counter()
    r = pipeline.permanent(a, jobs_at_least=args.jobs, leaf_order=args.leaf, measure_jobs=True,
                           leaf_budget_bytes=int(args.budget_gb * (1 << 30)))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    stages = {s: P.sperm_timing_get(s)[0] for s in ("expand", "kklll", "rnw_prep", "rnw", "rnw_finalize")}
    terms, fma, alu = P.sperm_rnw_stats(reset=True)
    xb, xn = P.sperm_expand_stats(reset=True)
    T = r.job_cycles.astype(np.float64)
    from scipy.stats import kendalltau
    out = {"workload": "per(C100), PAPER.md appendix graph", "per": str(r.value), "paper_table_T12_total": str(pin),
           "matches_paper": r.value == pin, "wall_s": wall, "jobs": r.num_jobs,
           "job_orders": {str(k): v for k, v in r.job_order_n.items()}, "leaf_order": args.leaf,
           "leaves": r.leaves, "terms": terms, "stage_ms": stages,
           "terms_per_s_rnw": terms / (stages["rnw"] * 1e-3) if stages["rnw"] else None,
           "expand_GBps": xb / (stages["expand"] * 1e-3) / 1e9 if stages["expand"] else None,
           "tau_T_estimate": float(kendalltau(T, r.estimates).statistic), "host": r.stats,
           "launches": P.sperm_launch_count(),
           "paper_T1_s_PentiumIII": 118413.21, "paper_T32_s_32xPentiumIII": 3796.85}
    print(json.dumps(out), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
