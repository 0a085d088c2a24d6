"""Writes tests/golden/oracle_values.txt: exact permanents of the workload graphs
computed ONLY by oracle/ (frontier DP and H_per), never by the CUDA path.

    python tools/make_golden.py [--fullerenes] [--n96]

Each line: <name> <value>   (name documents the workload recipe).
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.frontier import bfs_order, per_frontier  # noqa: E402
from oracle.hybrid import h_per  # noqa: E402
from workloads import dodecahedron, paper_graph, random_fullerene, truncated_icosahedron  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_values.txt")


def main():
    vals = {}
    if os.path.exists(OUT):
        for ln in open(OUT):
            if ln.strip() and not ln.startswith("#"):
                k, v = ln.split()
                vals[k] = v
    a = dodecahedron()
    vals["C20_dodecahedron"] = str(h_per(a))
    assert int(vals["C20_dodecahedron"]) == per_frontier(a)
    for name, g in (("C60_truncated_icosahedron", truncated_icosahedron()), ("C60_paper_appendix", paper_graph("C60"))):
        if name not in vals:
            vals[name] = str(per_frontier(g, bfs_order(g)))
    if "--fullerenes" in sys.argv:
        for n in (70, 76, 80, 84):
            for iso in range(4):
                key = f"fullerene_n{n}_seed2024_iso{iso}"
                if key in vals:
                    continue
                g, _ = random_fullerene(n, 2024, iso)
                t = time.time()
                vals[key] = str(per_frontier(g, bfs_order(g)))
                print(key, vals[key], f"{time.time() - t:.1f}s", flush=True)
                _write(vals)
    if "--n96" in sys.argv:
        # configs[4]: the spiral fullerene n=96 (isomer 0) and the random 3-regular n=96
        # (PCG64([2024, 96])), by the C frontier DP (oracle/frontier.c; ~2 and ~4 CPU-minutes)
        import numpy as np
        from oracle.cfrontier import narrow_order, per_frontier_c
        from workloads import random_3perm
        g, _ = random_fullerene(96, 2024, 0)
        rng = np.random.default_rng(np.random.PCG64([2024, 96]))
        r = random_3perm(96, rng)
        for key, m, order in (("fullerene_n96_seed2024_iso0", g, bfs_order(g)),
                              ("random3reg_n96_seed2024_96", r, narrow_order(r))):
            if key in vals:
                continue
            t = time.time()
            vals[key] = str(per_frontier_c(m, order))
            print(key, vals[key], f"{time.time() - t:.1f}s", flush=True)
            _write(vals)
    _write(vals)


def _write(vals):
    with open(OUT, "w") as f:
        f.write("# Exact permanents computed by oracle/ only (tools/make_golden.py); see DESIGN.md §6.\n")
        for k in sorted(vals):
            f.write(f"{k} {vals[k]}\n")


if __name__ == "__main__":
    main()
