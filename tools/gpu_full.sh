#!/bin/bash
# Evidence run: default bench (+clocks), reference arm, other configs, ncu launch list
# of our kernels for the default command, one --set full capture at full size.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_${TAG}.csv &
SMI=$!
python bench.py > gpurun_out/bench_default_${TAG}.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench_default_${TAG}.log
kill $SMI
python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.log 2>&1; echo "ref_rc=$?" >> gpurun_out/bench_ref_${TAG}.log
for cfg in 1 3 4 6 7; do python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_cfg${cfg}_${TAG}.log 2>&1; done
python bench.py --config 4 --kernel strip --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg4_fast_${TAG}.log 2>&1
python bench.py --kernel general --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg2_general_${TAG}.log 2>&1
python bench.py --out f16 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg2_f16_${TAG}.log 2>&1
python bench.py --config 3 --mode mean --filter fd --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg3_fdmean_${TAG}.log 2>&1
python bench.py --mode mean --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg2_mean_${TAG}.log 2>&1
python bench.py --layout packed --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg2_packed_${TAG}.log 2>&1
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
[ -z "$NO_NCU" ] && $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tfn_ --csv \
    --log-file gpurun_out/launches_default_${TAG}.csv $CMD > gpurun_out/ncu_launch_default_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tfn_strip -s 4 -c 1 \
    -o gpurun_out/prof_full_${TAG} -f $CMD > gpurun_out/ncu_full_default_${TAG}.log 2>&1
echo "ncu_rc=$?"
for f in gpurun_out/bench_*_${TAG}.log; do echo "$f: $(grep '^{' $f | python -c 'import json,sys
for l in sys.stdin:
    d=json.loads(l); print(round(d["value"]), d.get("roofline",{}).get("frac"), d.get("config",{}).get("workload","")[:60])')"; done
