"""GPU timeline of one whole-path run (torch.profiler / CUPTI kernel records): device busy time,
idle gaps and what precedes them, to locate host round-trip stalls in the pipeline.

    python tools/timeline.py --workload c100 --leaf 16 [--jobs 159] [--out gpurun_out/timeline.json]
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c100", choices=["c100", "c60", "fullerene96", "configs1"])
    ap.add_argument("--jobs", type=int, default=159)
    ap.add_argument("--leaf", type=int, default=16)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "timeline.json"))
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_1112_6072_b200 import pipeline
    from workloads import dodecahedron, paper_graph, random_fullerene
    if args.workload == "fullerene96":
        a, _ = random_fullerene(96, 2024, 0)
    elif args.workload == "configs1":
        a = None
    else:
        a = paper_graph("C100" if args.workload == "c100" else "C60")
    pipeline.permanent(dodecahedron(), jobs_at_least=8, leaf_order=12)
    torch.cuda.synchronize()
    if args.workload == "configs1":  # the bench step: one sperm_permanent over 256 n=24 matrices, x10
        import paper_1112_6072_b200 as P
        from workloads import random_3perm_batch
        mats = torch.tensor(random_3perm_batch(256, 24, 2024), dtype=torch.int32, device="cuda")
        for _ in range(3):
            P.sperm_permanent(mats, min_primes=1)
        torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        if args.workload == "configs1":
            for _ in range(10):
                res, k = P.sperm_permanent(mats, min_primes=1)

            class _R:
                value = "configs1 x10"
            r = _R()
        else:
            r = pipeline.permanent(a, jobs_at_least=args.jobs, leaf_order=args.leaf)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    ev = []
    for e in prof.events():
        if e.device_type.name == "CUDA" and e.time_range.end > e.time_range.start:
            ev.append((e.time_range.start, e.time_range.end, e.name))
    ev.sort()
    busy = 0.0
    gaps = []
    cur_s, cur_e, cur_name = None, None, None
    by_kernel = collections.defaultdict(float)
    for s, e, name in ev:
        by_kernel[name[:60]] += e - s
        if cur_e is None:
            cur_s, cur_e, cur_name = s, e, name
            continue
        if s > cur_e:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, cur_name[:50], name[:50]))
            cur_s, cur_e, cur_name = s, e, name
        elif e > cur_e:
            cur_e, cur_name = e, name
    if cur_e is not None:
        busy += cur_e - cur_s
    span = (ev[-1][1] - ev[0][0]) if ev else 0.0
    gap_by = collections.defaultdict(lambda: [0, 0.0])
    for g, p, nx in gaps:
        k = f"{p} -> {nx}"
        gap_by[k][0] += 1
        gap_by[k][1] += g
    top = sorted(gap_by.items(), key=lambda kv: -kv[1][1])[:15]
    out = {"workload": args.workload, "per": str(r.value), "wall_s": wall, "span_s": span * 1e-6,
           "busy_s": busy * 1e-6, "idle_s": (span - busy) * 1e-6, "gaps": len(gaps),
           "top_gaps": [{"between": k, "count": c, "total_ms": t * 1e-3} for k, (c, t) in top],
           "kernel_ms": {k: v * 1e-3 for k, v in sorted(by_kernel.items(), key=lambda kv: -kv[1])[:20]}}
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
