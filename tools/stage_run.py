"""Whole-path run of one workload with per-stage device timings (the library's CUDA-event
timers) and the expansion's algorithmic GB/s.  The pipeline runs every stage on one stream
(unless SPERM_PIPELINE_OVERLAP=1), so the stage timings add up to the device time.

    python tools/stage_run.py --workload fullerene96 --jobs 1000 --leaf 20
    python tools/stage_run.py --workload c100 --jobs 159 --leaf 16
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
    ap.add_argument("--workload", default="fullerene96", choices=["fullerene96", "random96", "c100", "c60"])
    ap.add_argument("--jobs", type=int, default=1000)
    ap.add_argument("--leaf", type=int, default=20)
    ap.add_argument("--seed", type=int, default=2024)
    args = ap.parse_args()
    import torch
    import paper_1112_6072_b200 as P
    from paper_1112_6072_b200 import pipeline
    import numpy as np
    from workloads import dodecahedron, paper_graph, random_fullerene, random_3perm
    if args.workload == "fullerene96":
        a, _ = random_fullerene(96, args.seed, 0)
    elif args.workload == "random96":
        a = random_3perm(96, np.random.Generator(np.random.PCG64([args.seed, 96])))
    else:
        a = paper_graph("C100" if args.workload == "c100" else "C60")
    pipeline.permanent(dodecahedron(), jobs_at_least=8, leaf_order=12)  # warm-up
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    P.sperm_expand_stats(reset=True)
    P.sperm_rnw_stats(reset=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = pipeline.permanent(a, jobs_at_least=args.jobs, leaf_order=args.leaf)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    st = {s: round(P.sperm_timing_get(s)[0], 1) for s in ("expand", "kklll", "rnw_prep", "rnw", "rnw_finalize")}
    xb, _ = P.sperm_expand_stats(reset=True)
    terms, _, _ = P.sperm_rnw_stats(reset=True)
    print(json.dumps({"workload": args.workload, "per": str(r.value), "wall_s": round(wall, 2), "jobs": r.num_jobs,
                      "leaves": r.leaves, "stage_ms": st,
                      "expand_GBps": round(xb / (st["expand"] * 1e-3) / 1e9, 1) if st["expand"] else None,
                      "terms_per_s_rnw": terms / (st["rnw"] * 1e-3) if st["rnw"] else None,
                      "overlap": os.environ.get("SPERM_PIPELINE_OVERLAP", "0")}), flush=True)


if __name__ == "__main__":
    main()
