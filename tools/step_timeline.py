"""Kernel-level timeline of the configs[1] bench step (torch.profiler / CUPTI records): every
kernel of a few steps, start and end relative to the step's first kernel, to see where the
step's time outside the R-NW kernels goes (prep, grouping, finalize, gaps).

    python tools/step_timeline.py [--steps 4] [--out gpurun_out/step_timeline.txt]
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "step_timeline.txt"))
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_1112_6072_b200 as P
    from workloads import random_3perm_batch
    mats = torch.tensor(random_3perm_batch(256, 24, 2024), dtype=torch.int32, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
    for _ in range(5):
        P.sperm_permanent(mats, min_primes=1)
    torch.cuda.synchronize()
    marks = []
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(args.steps):
            flush.fill_(i)
            torch.cuda.synchronize()
            P.sperm_permanent(mats, min_primes=1)
            torch.cuda.synchronize()
    ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                if e.device_type.name == "CUDA" and e.time_range.end > e.time_range.start)
    lines = []
    step, t0 = -1, None
    for s, e, name in ev:
        if "Fill" in name or "fill" in name:
            step += 1
            t0 = None
            lines.append(f"--- step {step}")
            continue
        if t0 is None:
            t0 = s
        lines.append(f"{(s - t0):9.2f} {(e - t0):9.2f} {(e - s):8.2f}  {name[:90]}")
    txt = "\n".join(lines)
    print(txt)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        f.write("# start_us end_us dur_us kernel (relative to the step's first kernel)\n" + txt + "\n")


if __name__ == "__main__":
    main()
