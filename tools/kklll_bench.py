"""KKLLL job weights (sperm_estimate) of a whole-path job list, timed alone (library timer),
optionally under ncu (the estimate calls are bracketed by cudaProfilerStart/Stop).

    python tools/kklll_bench.py [--workload fullerene96] [--jobs 1000] [--trials 0]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="fullerene96", choices=["fullerene96", "c100", "c60", "c20"])
    ap.add_argument("--jobs", type=int, default=1000)
    ap.add_argument("--trials", type=int, default=0)
    ap.add_argument("--limit", type=int, default=0, help="estimate only the first LIMIT jobs of each order")
    args = ap.parse_args()
    import torch
    import paper_1112_6072_b200 as P
    from paper_1112_6072_b200 import pipeline
    from workloads import dodecahedron, paper_graph, random_fullerene, truncated_icosahedron
    a = (random_fullerene(96, 2024, 0)[0] if args.workload == "fullerene96" else
         truncated_icosahedron() if args.workload == "c60" else
         dodecahedron() if args.workload == "c20" else paper_graph("C100"))
    sets = pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=args.jobs)
    if args.limit:
        sets = [pipeline.NodeSet(s.n, s.mats[:args.limit], s.coef[:args.limit], s.job[:args.limit]) for s in sets]
    P.sperm_estimate(sets[0].mats[:1], trials=4, ids=sets[0].job[:1])  # warm-up
    torch.cuda.synchronize()
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    torch.cuda.profiler.start()
    est = [P.sperm_estimate(s.mats, trials=args.trials, seed=1, ids=s.job) for s in sets]
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ms, _ = P.sperm_timing_get("kklll")
    orders = {s.n: s.count for s in sets}
    trials = {s.n: (args.trials or s.n * s.n) for s in sets}
    lu_ops = sum(s.count * trials[s.n] * 8.0 * sum((s.n - k - 1) ** 2 for k in range(s.n)) for s in sets)
    print(json.dumps({"workload": args.workload, "orders": orders, "trials": trials, "kklll_ms": ms,
                      "fp64_update_ops": lu_ops, "fp64_Gops": lu_ops / (ms * 1e-3) / 1e9,
                      "checksum": float(sum(float(e.sum()) for e in est))}))


if __name__ == "__main__":
    main()
