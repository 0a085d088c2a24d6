"""per(C60) by the whole path (configs[2]: J >= 992, L = 32) with the second run bracketed by
cudaProfilerStart/Stop, for ncu captures of its kernels:

    ncu --set full --import-source on --profile-from-start off -k regex:rnw_tree -o /tmp/c60 python tools/c60_probe.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1112_6072_b200 as P
    from paper_1112_6072_b200 import pipeline
    from workloads import truncated_icosahedron
    a = truncated_icosahedron()
    pipeline.permanent(a, jobs_at_least=992, leaf_order=32)
    torch.cuda.synchronize()
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    torch.cuda.profiler.start()
    t = time.perf_counter()
    r = pipeline.permanent(a, jobs_at_least=992, leaf_order=32)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    torch.cuda.profiler.stop()
    st = {s: round(P.sperm_timing_get(s)[0], 3) for s in ("expand", "kklll", "rnw_prep", "rnw", "rnw_finalize")}
    print(r.value, round(wall * 1e3, 2), "ms", st, {k: v for k, v in os.environ.items() if k.startswith("SPERM_")})


if __name__ == "__main__":
    main()
