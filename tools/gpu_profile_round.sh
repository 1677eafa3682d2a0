#!/bin/bash
# ncu evidence for the round: for each config, a plain bench run (must exit 0), the launch
# list (gpu__time_duration per launch) and one --set full capture of the strip kernel.
#   TAG=r01d CONFIGS="2 6" tools/gpu_profile_round.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
for cfg in ${CONFIGS:-2}; do
  CMD="python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-e2e"
  $CMD > gpurun_out/${TAG}_plain_config$cfg.json 2> gpurun_out/${TAG}_plain_config$cfg.err || { echo "plain config $cfg failed"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches_config$cfg.csv $CMD > /dev/null 2>&1
  echo "launches config $cfg rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:tfn_strip -s 4 -c 1 \
      -o gpurun_out/${TAG}_strip_config$cfg -f $CMD > gpurun_out/${TAG}_ncu_full_config$cfg.log 2>&1
  echo "full config $cfg rc=$?"
done
