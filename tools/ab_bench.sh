#!/bin/bash
# A-B of library variants on the configs[1] bench line (tools/build_variant.py builds them).
#   bash tools/ab_bench.sh [variant ...]      (default: the main build + every variants/*.so)
cd "$(dirname "$0")/.."
libs=("$@")
[ ${#libs[@]} -eq 0 ] && libs=(main $(ls paper_1112_6072_b200/variants/*.so 2>/dev/null | sed 's#.*/libsperm_##; s#\.so##'))
for rep in 1 2; do
  for v in "${libs[@]}"; do
    if [ "$v" = main ]; then unset SPERM_LIB; else export SPERM_LIB=paper_1112_6072_b200/variants/libsperm_$v.so; fi
    python bench.py --no-ph --no-c100 --no-strong --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$v', 'value %.4g' % d['value'], 'step %.4f' % d['ms_per_step'], 'kernel %.4f' % d['roofline']['kernel_ms_per_step'],
      'nospec %.4f' % d['without_speculation']['ms_per_step'], 'e2e %.4g' % d['e2e']['value'])"
  done
done
