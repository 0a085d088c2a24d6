"""configs[3]: per(A) of the 16 seeded spiral fullerenes (n in {70,76,80,84}, 4 isomers each) by
the whole path on one GPU, checked against the oracle's frontier-DP values
(tests/golden/oracle_values.txt, written by tools/make_golden.py from oracle/ only).

    python tools/fullerene_run.py [--leaf 16] [--jobs 256] [--out gpurun_out/fullerenes.json]
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
    ap.add_argument("--leaf", type=int, default=16)
    ap.add_argument("--jobs", type=int, default=256)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "fullerenes.json"))
    args = ap.parse_args()
    import torch
    from paper_1112_6072_b200 import pipeline
    from workloads import dodecahedron, random_fullerene
    gold = {}
    for ln in open(os.path.join(ROOT, "tests", "golden", "oracle_values.txt")):
        if ln.strip() and not ln.startswith("#"):
            k, v = ln.split()
            gold[k] = int(v)
    pipeline.permanent(dodecahedron(), jobs_at_least=8, leaf_order=12)  # warm-up
    rows = []
    for n in (70, 76, 80, 84):
        for iso in range(4):
            a, pent = random_fullerene(n, 2024, iso)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = pipeline.permanent(a, jobs_at_least=args.jobs, leaf_order=args.leaf)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            key = f"fullerene_n{n}_seed2024_iso{iso}"
            rows.append({"n": n, "isomer": iso, "pentagons": pent, "per": str(r.value),
                         "oracle": str(gold.get(key)), "match": gold.get(key) == r.value, "wall_s": wall,
                         "jobs": r.num_jobs, "leaves": r.leaves, "terms": r.terms})
            print(json.dumps(rows[-1]), flush=True)
    out = {"leaf_order": args.leaf, "jobs_at_least": args.jobs, "all_match": all(x["match"] for x in rows),
           "total_wall_s": sum(x["wall_s"] for x in rows), "runs": rows}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "runs"}))


if __name__ == "__main__":
    main()
