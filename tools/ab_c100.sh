cd $GRAFT_REPO_ROOT
for env in "SPERM_EXPAND_ORDERED=1" "SPERM_EXPAND_ORDERED=0" "SPERM_EXPAND_ORDERED=1" "SPERM_EXPAND_ORDERED=0"; do
env $env python - <<'PY'
import sys, time, os
sys.path.insert(0, '.')
import torch
import paper_1112_6072_b200 as P
from paper_1112_6072_b200 import pipeline
from workloads import paper_graph, dodecahedron
pipeline.permanent(dodecahedron(), jobs_at_least=8, leaf_order=12)
P.sperm_timing_enable(True); P.sperm_timing_reset()
torch.cuda.synchronize(); t = time.perf_counter()
r = pipeline.permanent(paper_graph("C100"), jobs_at_least=159, leaf_order=15)
torch.cuda.synchronize()
st = {s: round(P.sperm_timing_get(s)[0]) for s in ("expand", "kklll", "rnw_prep", "rnw", "rnw_finalize")}
print(os.environ.get("SPERM_EXPAND_ORDERED"), r.value, round(time.perf_counter() - t, 2), st, flush=True)
PY
done
