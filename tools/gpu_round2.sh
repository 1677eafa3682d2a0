#!/bin/bash
# Round-2 measurement batch (one gpurun call): the driver's default bench line, the other
# configs, the Table II counterpart (4 filters x mean/median on configs[1]), the fp32 kernel
# on the same workload, then the ncu launch list + one --set full capture of the default run.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-r02}
python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "default rc=$?"
for cfg in 3 4 6 7; do
  python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu > gpurun_out/${T}_bench_config$cfg.json 2>&1; echo "config $cfg rc=$?"
done
for f in fd sobel scharr prewitt; do for m in mean median; do
  python bench.py --filter $f --mode $m --steps 20 --warmup 3 --no-cpu --no-e2e | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'filter':'$f','mode':'$m','Gpx_s':d['value']/1e3,'fps':d['config']['fps'],'frac':d['roofline']['frac'],'launch_ms':d['roofline']['launch_ms'],'clocks':d['clocks']}))"
done; done > gpurun_out/${T}_table2_sweep.jsonl 2>&1; echo "sweep rc=$?"
python bench.py --kernel f32 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_f32kernel.json 2>&1; echo "f32 rc=$?"
CMD="python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/${T}_plain_config2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_config2.csv $CMD > /dev/null 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/${T}_plain2_config2.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tfn_strip -s 4 -c 1 -o gpurun_out/${T}_strip_config2 -f $CMD > gpurun_out/${T}_ncu_full_config2.log 2>&1
echo "full rc=$?"
