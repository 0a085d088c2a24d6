#!/bin/bash
# A-B of library variants (tools/build_variant.py) on fixed C100 leaf sets of order 15 and 16.
#   bash tools/ab_leaf.sh [variant ...]
cd "$(dirname "$0")/.."
libs=("$@"); [ ${#libs[@]} -eq 0 ] && libs=(main)
for rep in 1 2; do
for v in "${libs[@]}"; do
  if [ "$v" = main ]; then unset SPERM_LIB; else export SPERM_LIB=paper_1112_6072_b200/variants/libsperm_$v.so; fi
  for L in 15 16; do
  python tools/leafbench.py --graph C100 --leaf $L --max-leaves $((L == 15 ? 4000000 : 2000000)) 2>&1 | tail -n 1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v L$L rnw %.2f prep %.2f fin %.2f ms' % (d['stage_ms']['rnw'], d['stage_ms']['rnw_prep'], d['stage_ms']['rnw_finalize']))"
  done
done; done
