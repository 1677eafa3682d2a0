#!/bin/bash
# Round-end style evidence: default bench, reference arm, ncu launch list of the
# default command, one --set full capture of the strip kernel.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_${TAG}.csv &
SMI=$!
python bench.py > gpurun_out/bench_default_${TAG}.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench_default_${TAG}.log
kill $SMI
python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.log 2>&1; echo "ref_rc=$?" >> gpurun_out/bench_ref_${TAG}.log
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_default_${TAG}.csv $CMD > gpurun_out/ncu_launch_default_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tfn_strip -s 4 -c 1 \
    -o gpurun_out/prof_full_${TAG} -f $CMD > gpurun_out/ncu_full_default_${TAG}.log 2>&1
echo "ncu_rc=$?"
tail -2 gpurun_out/bench_default_${TAG}.log | cut -c1-300; tail -2 gpurun_out/bench_ref_${TAG}.log | cut -c1-300
