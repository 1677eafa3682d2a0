#!/bin/bash
# End-of-round measurement batch (one gpurun call): smoke, the GPU test suite, the driver's
# default bench line, every other config, the Table II counterpart sweep (4 filters x
# mean/median on configs[1]) and the ncu launch list of the default run.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-r02c}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; echo "smoke rc=$?"
python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gputests.txt 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/${T}_gputests.txt
python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "default rc=$?"
for cfg in 1 3 4 5 6 7; do
  python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu > gpurun_out/${T}_bench_config$cfg.json 2>&1; echo "config $cfg rc=$?"
done
for f in fd sobel scharr prewitt; do for m in mean median; do
  python bench.py --filter $f --mode $m --steps 20 --warmup 3 --no-cpu --no-e2e | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'filter':'$f','mode':'$m','Gpx_s':d['value']/1e3,'fps':d['config']['fps'],'frac':d['roofline']['frac'],'launch_ms':d['roofline']['launch_ms'],'clocks':d['clocks']}))"
done; done > gpurun_out/${T}_table2_sweep.jsonl 2>&1; echo "sweep rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_reference.json 2>&1; echo "reference rc=$?"
CMD="python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/${T}_plain_config2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_config2.csv $CMD > /dev/null 2>&1
echo "launches rc=$?"
