"""Timing probe of sperm_expand_subtree on C100 nodes (the paper's case study): PH jobs
(J >= 159) of job 0.. expanded level by level to order n0, then up to --roots of those nodes
expanded depth first to leaves of order L, `--reps` times (library event timers).

    python tools/subtree_probe.py --leaf 15 --n0 27 --roots 200000
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
    ap.add_argument("--leaf", type=int, default=15)
    ap.add_argument("--n0", type=int, default=27)
    ap.add_argument("--roots", type=int, default=200000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--workload", default="c100", choices=["c100", "fullerene96"])
    args = ap.parse_args()
    import torch
    import paper_1112_6072_b200 as P
    from paper_1112_6072_b200 import pipeline
    from workloads import paper_graph, random_fullerene
    a = paper_graph("C100") if args.workload == "c100" else random_fullerene(96, 2024, 0)[0]
    jobs = pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=159)[0]
    lv = None
    for j in range(jobs.count):
        one = pipeline.NodeSet(jobs.n, jobs.mats[j:j + 1], jobs.coef[j:j + 1], jobs.job[j:j + 1])
        s = pipeline.expand_to_leaves(one, args.n0)[0]
        lv = s if lv is None else pipeline.NodeSet(s.n, torch.cat([lv.mats, s.mats]), torch.cat([lv.coef, s.coef]),
                                                   torch.cat([lv.job, s.job]))
        if lv.count >= args.roots:
            break
    k = min(lv.count, args.roots)
    mats, coef, job = lv.mats[:k].contiguous(), lv.coef[:k].contiguous(), lv.job[:k].contiguous()
    cap = 64 * k
    r = P.sperm_expand_subtree(mats, args.leaf, cap, coef, job)  # warm-up
    nleaves = r[0][0].shape[0]
    del r
    torch.cuda.synchronize()
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    P.sperm_expand_subtree_stats(reset=True)
    for _ in range(args.reps):
        r = P.sperm_expand_subtree(mats, args.leaf, cap, coef, job)
        del r
    torch.cuda.synchronize()
    ms, launches = P.sperm_timing_get("expand")
    nbytes, roots = P.sperm_expand_subtree_stats(reset=True)
    P.sperm_timing_enable(False)
    print(json.dumps({"workload": args.workload, "n0": lv.n, "L": args.leaf, "roots": k, "leaves": nleaves,
                      "ms_per_call": ms / args.reps, "leaves_per_s": nleaves * args.reps / (ms * 1e-3),
                      "GBps_algorithmic": nbytes / (ms * 1e-3) / 1e9,
                      "env": {e: os.environ[e] for e in os.environ if e.startswith("SPERM_")}}), flush=True)


if __name__ == "__main__":
    main()
