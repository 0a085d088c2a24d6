"""One Eq. (2) expansion level (sperm_expand) of C100 descendants at a small order, timed with
the library's event timers — the shape that dominates the whole-path expansion at L = 16.

    python tools/expand_level.py [--order 20] [--nodes 2000000] [--reps 5]
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
    ap.add_argument("--order", type=int, default=20)
    ap.add_argument("--nodes", type=int, default=2_000_000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_1112_6072_b200 as P
    from paper_1112_6072_b200 import pipeline
    from workloads import paper_graph
    top = pipeline.pre_expand(pipeline.root_nodeset(paper_graph("C100")), jobs_at_least=200_000)[0]
    take = 64
    while True:  # grow the seed set until its descendants at `order` reach `nodes`
        seed = pipeline.NodeSet(top.n, top.mats[:take], top.coef[:take], top.job[:take])
        sets = pipeline.expand_to_leaves(seed, args.order)
        lvl = [s for s in sets if s.n == args.order]
        cnt = lvl[0].count if lvl else 0
        if cnt >= args.nodes or take >= top.count:
            break
        take = min(top.count, take * 2)
    s = lvl[0]
    s = pipeline.NodeSet(s.n, s.mats[:args.nodes], s.coef[:args.nodes], s.job[:args.nodes])
    P.sperm_expand(s.mats, s.coef, s.job)
    torch.cuda.synchronize()
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    P.sperm_expand_stats(reset=True)
    torch.cuda.profiler.start()  # ncu --profile-from-start off captures only these levels
    for _ in range(args.reps):
        P.sperm_expand(s.mats, s.coef, s.job)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ms, launches = P.sperm_timing_get("expand")
    nbytes, nodes = P.sperm_expand_stats(reset=True)
    print(json.dumps({"order": s.n, "nodes": s.count, "ms_per_level": ms / args.reps,
                      "GBps": nbytes / (ms * 1e-3) / 1e9, "bytes_per_level": nbytes / args.reps}))


if __name__ == "__main__":
    main()
