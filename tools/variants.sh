#!/bin/bash
# Throughput of the strip kernel variants (fast / general / adaptive) on configs 2, 3, 4:
#   tools/variants.sh [lib]   (TFN_LIB, default the in-tree library)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
LIB=${1:-paper_2005_08165_b200/libtfn.so}
for cfg in 2 3 4; do
  for k in strip general adaptive; do
    TFN_LIB=$LIB python bench.py --config $cfg --kernel $k --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('config $cfg $k', round(d['value']), round(d['roofline']['frac'],4))
"
  done
done
