#!/bin/bash
# Strip-height / grid sweep of the strip kernel on one config (runtime options, no rebuild):
#   CONFIG=2 tools/sweep_strip.sh > gpurun_out/sweep.txt
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for rep in 1 2; do
  for sh in ${STRIP_HS:-24 32 48 64 96 160}; do
    python bench.py --config ${CONFIG:-2} --steps 30 --warmup 5 --no-cpu --no-e2e --strip-h $sh ${SWEEP_ARGS} 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('strip_h=$sh', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['config'].get('kernel_variant'))
"
  done
done
