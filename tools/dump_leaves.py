"""Dump a sample of leaves of a whole-path run (for offline plan studies on the CPU).

    python tools/dump_leaves.py --workload c100 --leaf 15 --count 4000 --out gpurun_out/leaves.npy
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c100", choices=["c100", "fullerene96"])
    ap.add_argument("--leaf", type=int, default=15)
    ap.add_argument("--count", type=int, default=4000)
    ap.add_argument("--out", default="gpurun_out/leaves.npy")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_1112_6072_b200 import pipeline
    from workloads import paper_graph, random_fullerene
    a = paper_graph("C100") if args.workload == "c100" else random_fullerene(96, 2024, 0)[0]
    jobs = pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=159)[0]
    rng = np.random.default_rng(1)
    pick = rng.choice(jobs.count, size=4, replace=False)
    out = []
    for j in pick:
        one = pipeline.NodeSet(jobs.n, jobs.mats[j:j + 1], jobs.coef[j:j + 1], jobs.job[j:j + 1])
        for lv in pipeline.iter_leaves(one, args.leaf):
            if lv.n == args.leaf:
                k = min(lv.count, args.count // 4)
                idx = torch.tensor(rng.choice(lv.count, size=k, replace=False), device=lv.mats.device)
                out.append(lv.mats.index_select(0, idx).cpu().numpy())
                break
    np.save(args.out, np.concatenate(out))
    print("dumped", sum(o.shape[0] for o in out))


if __name__ == "__main__":
    main()
