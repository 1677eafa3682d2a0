#!/bin/bash
# ncu evidence for the strip kernel: plain run first (must exit 0), then the launch
# list and one --set full capture.  Usage: PROF_ARGS="--config 2" tools/gpu_profile.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
CMD="python bench.py --profile --frames ${FRAMES:-256} --steps 3 --warmup 2 ${PROF_ARGS}"
$CMD > gpurun_out/prof_plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tfn_ --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tfn_strip -s 2 -c 1 \
    -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "profile_rc=$?"
tail -3 gpurun_out/prof_plain_${TAG}.log
