"""Micro-benchmark of sperm_permanent on a fixed leaf set (device timers per stage).

    python tools/leafbench.py [--graph C100] [--jobs 200000] [--leaf 16] [--max-leaves 4000000]

Expands the appendix graph (PH Step 2 to >= J jobs, then H_per to order <= L), keeps up to
--max-leaves leaves of the leaf order, and times rnw_prep / rnw / rnw_finalize of one
sperm_permanent call over them (after a warm-up call), single stream."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graph", default="C100")
    ap.add_argument("--jobs", type=int, default=2000)
    ap.add_argument("--leaf", type=int, default=16)
    ap.add_argument("--max-leaves", type=int, default=4_000_000)
    args = ap.parse_args()
    import torch
    import paper_1112_6072_b200 as P
    from paper_1112_6072_b200 import pipeline
    from workloads import paper_graph
    a = paper_graph(args.graph)
    sets = pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=args.jobs)
    js = sets[0]
    js = pipeline.NodeSet(js.n, js.mats[:64], js.coef[:64], js.job[:64])
    leaves = None
    for lv in pipeline.iter_leaves(js, args.leaf):
        if lv.n == args.leaf:
            leaves = lv if leaves is None else pipeline.NodeSet(lv.n, torch.cat([leaves.mats, lv.mats]),
                                                                torch.cat([leaves.coef, lv.coef]),
                                                                torch.cat([leaves.job, lv.job]))
            if leaves.count >= args.max_leaves:
                break
    m = leaves.mats[:args.max_leaves].contiguous()
    c = leaves.coef[:args.max_leaves].contiguous()
    P.sperm_permanent(m, coef=c, min_primes=3, max_primes=3)  # warm-up
    torch.cuda.synchronize()
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    P.sperm_rnw_stats(reset=True)
    t0 = time.perf_counter()
    torch.cuda.profiler.start()  # ncu --profile-from-start off captures only this call
    P.sperm_permanent(m, coef=c, min_primes=3, max_primes=3)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    wall = time.perf_counter() - t0
    st = {s: P.sperm_timing_get(s)[0] for s in ("rnw_prep", "rnw", "rnw_finalize")}
    terms = P.sperm_rnw_stats(reset=True)[0]
    print(json.dumps({"leaves": int(m.shape[0]), "n": int(m.shape[1]), "wall_ms": wall * 1e3, "stage_ms": st,
                      "prep_ns_per_leaf": st["rnw_prep"] * 1e6 / m.shape[0],
                      "terms_per_s_rnw": terms / (st["rnw"] * 1e-3)}))


if __name__ == "__main__":
    main()
