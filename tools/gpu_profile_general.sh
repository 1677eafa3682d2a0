#!/bin/bash
# ncu evidence for the general strip variant (config 4, AUTO -> general): launch list of
# the bench command, then one --set full capture of a general-variant launch.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
CMD="python bench.py --config 4 --kernel general --steps 4 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/plain_general_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tfn_strip -s 4 -c 1 \
    -o gpurun_out/prof_general_${TAG} -f $CMD > gpurun_out/ncu_general_${TAG}.log 2>&1
echo "ncu_rc=$?"
tail -2 gpurun_out/plain_general_${TAG}.log | cut -c1-200
