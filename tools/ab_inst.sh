#!/bin/bash
# instructions per pixel + duration of one config-2 strip launch per library variant (ncu, one GPU):
#   tools/ab_inst.sh abl/lib_a.so abl/lib_b.so ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for lib in "$@"; do
  TFN_LIB=$lib ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,launch__registers_per_thread \
      --clock-control none -k regex:tfn_strip -s 2 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e ${AB_ARGS} 2>/dev/null \
    | python tools/ncu_csv_inst.py "$lib"
done
