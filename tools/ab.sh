#!/bin/bash
# A/B throughput of library variants on the same box: tools/ab.sh libA.so libB.so ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in "$@"; do
    TFN_LIB=$lib python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e ${AB_ARGS} 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$lib', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])
"
  done
done
