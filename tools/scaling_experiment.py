"""Load-balance study of configs[4] (BASELINE.json): the paper's scheduling comparison
(§4, Tables 5-7: natural vs exact-time vs estimated order) on B200-measured job costs.

    python tools/scaling_experiment.py [--jobs 2000] [--leaf 22] [--out gpurun_out/scaling.json]

Workload: a seeded n=96 3-regular 0/1 matrix (union of three disjoint random permutation
matrices) and a seeded n=96 spiral fullerene (reading of configs[4] budgeted as in
SURVEY F6: >= J jobs from the PH pre-expansion, leaves of order <= L).  One GPU runs the whole
PH path with per-leaf SM-cycle counters (sperm_permanent d_leaf_cycles), which give every
job's measured cost T_i.  For G in {1,2,4,8} GPUs and each ordering policy the script then
reports the parallel efficiency sum(T) / (G * makespan) of
  * static:  the plan sperm_schedule makes from the policy's planned weights (what the
             multi-GPU run deals to the ranks; estimate = LPT on KKLLL estimates, S1), and
  * dynamic: list scheduling in the policy's order with the actual costs (a job goes to the
             GPU that frees first — the paper's Step 3 semantics),
plus Kendall tau(T, estimate) and tau(T, size).  Costs are SM cycles, so
the efficiencies do not depend on how many GPUs measured them.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def dynamic_ls(order, cost, G):
    loads = np.zeros(G)
    for j in order:
        g = int(np.argmin(loads))
        loads[g] += cost[j]
    return loads.max()


def static_plan(P, weights, cost, G, policy, seed=7):
    mach, order, _ = P.sperm_schedule(weights, G, policy, seed=seed)
    loads = np.bincount(mach, weights=cost, minlength=G)
    return loads.max(), order


def kendall_tau(x, y):
    from scipy.stats import kendalltau
    return float(kendalltau(x, y).statistic)


def study(P, pipeline, name, a, J, L, Gs=(1, 2, 4, 8)):
    import torch
    # device time of the replicated pre-expansion alone (every rank repeats it)
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    pipeline.pre_expand(pipeline.root_nodeset(a), jobs_at_least=J)
    torch.cuda.synchronize()
    pre_ms = P.sperm_timing_get("expand")[0]
    P.sperm_timing_reset()
    t0 = time.perf_counter()
    r = pipeline.permanent(a, jobs_at_least=J, leaf_order=L, measure_jobs=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    stage_ms = {s: P.sperm_timing_get(s)[0] for s in ("expand", "kklll", "rnw_prep", "rnw", "rnw_finalize")}
    P.sperm_timing_enable(False)
    T = r.job_cycles.astype(np.float64)
    est = r.estimates
    size = r.job_sizes.astype(np.float64)
    rng = np.random.default_rng(11)
    res = {"workload": name, "n": int(a.shape[0]), "per": str(r.value), "jobs": r.num_jobs, "leaves": r.leaves,
           "terms": r.terms, "wall_s_1gpu": wall, "stage_ms": stage_ms,
           "job_orders": {str(k): v for k, v in r.job_order_n.items()},
           "tau_T_estimate": kendall_tau(T, est), "tau_T_size": kendall_tau(T, size),
           "cost_cv": float(T.std() / T.mean()), "efficiency": {}}
    total = T.sum()
    policies = {
        "natural": (np.ones_like(T), "natural", np.arange(len(T))),
        "random": (np.ones_like(T), "random", rng.permutation(len(T))),
        "size": (size, "estimate", np.argsort(-size, kind="stable")),
        "estimate": (est, "estimate", np.argsort(-est, kind="stable")),
        "exact": (T, "estimate", np.argsort(-T, kind="stable")),
    }
    # projected whole-path efficiency on G GPUs from the measured single-GPU stage times: the
    # pre-expansion is replicated, KKLLL sharded (1/G), the per-job work (expansion to leaves,
    # prep, R-NW, finalize) split as the static plan deals the measured job costs T_i
    kk_s = stage_ms["kklll"] * 1e-3
    pre_s = pre_ms * 1e-3
    eval_s = (stage_ms["expand"] - pre_ms + stage_ms["rnw_prep"] + stage_ms["rnw"] + stage_ms["rnw_finalize"]) * 1e-3
    t1 = pre_s + kk_s + eval_s
    res["projection"] = {"pre_expand_s": pre_s, "kklll_s": kk_s, "per_job_work_s": eval_s, "by_G": {}}
    for G in Gs:
        row = {}
        proj = {}
        for pname, (w, code, dyn_order) in policies.items():
            ms_static, _ = static_plan(P, w, T, G, code)
            ms_dyn = dynamic_ls(dyn_order, T, G)
            row[pname] = {"static": total / (G * ms_static), "dynamic": total / (G * ms_dyn)}
            tg = pre_s + kk_s / G + eval_s * ms_static / total
            proj[pname] = {"wall_s": tg, "efficiency": t1 / (G * tg)}
        res["efficiency"][str(G)] = row
        res["projection"]["by_G"][str(G)] = proj
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", default="48,160,1000", help="comma-separated J values (jobs_at_least)")
    ap.add_argument("--leaf", type=int, default=16)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "scaling.json"))
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    import paper_1112_6072_b200 as P
    from paper_1112_6072_b200 import pipeline
    from workloads import random_3perm, random_fullerene
    rng = np.random.default_rng(np.random.PCG64([2024, 96]))
    mats = [("random 3-regular n=96 (seed [2024,96])", random_3perm(96, rng)),
            ("spiral fullerene n=96 (seed 2024, isomer 0)", random_fullerene(96, 2024, 0)[0])]
    out = {"jobs_at_least": args.jobs, "leaf_order": args.leaf, "studies": []}
    for J in [int(x) for x in args.jobs.split(",")]:
        for name, a in mats:
            res = study(P, pipeline, name, a, J, args.leaf)
            res["jobs_at_least"] = J
            out["studies"].append(res)
            print(json.dumps({k: v for k, v in res.items() if k != "efficiency"}), flush=True)
            for G, row in res["efficiency"].items():
                print(f"  G={G}: " + "  ".join(f"{p}: s{v['static']:.4f}/d{v['dynamic']:.4f}"
                                               for p, v in row.items()), flush=True)
                pr = res["projection"]["by_G"][G]
                print(f"  G={G} projected whole-path efficiency: " +
                      "  ".join(f"{p}: {v['efficiency']:.3f}" for p, v in pr.items()), flush=True)
            with open(args.out, "w") as f:
                json.dump(out, f, indent=1)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
