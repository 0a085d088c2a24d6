import os, sys, json
sys.path.insert(0, '.')
import torch, numpy as np
import paper_1112_6072_b200 as P
from workloads import random_3perm_batch
for n in (12, 16, 20, 24, 27):
    mats = torch.tensor(random_3perm_batch(2000, n, seed=5), dtype=torch.int32, device='cuda')
    out = {}
    for wm in ("99", "1"):
        os.environ["SPERM_KKLLL_WARP_MIN"] = wm
        P.sperm_estimate(mats[:4], trials=4)
        torch.cuda.synchronize()
        P.sperm_timing_enable(True); P.sperm_timing_reset()
        e = P.sperm_estimate(mats, trials=0, seed=1)
        torch.cuda.synchronize()
        out[wm] = (round(P.sperm_timing_get("kklll")[0], 3), float(e.sum()))
    print(n, out, flush=True)
