#!/bin/bash
# configs[2] (disparity: FD / Scharr x mean / median) and configs[3] at both sizes it names
# (1080x1920 x128 and 2160x3840 x32, holes + salt, Prewitt + median): one JSON summary line each
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() {
  python bench.py "$@" --steps 20 --warmup 3 --no-cpu --no-e2e | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print(json.dumps({'args': '$*', 'workload': c['workload'], 'filter': c['filter'], 'mode': c['nz_mode'], 'H': c['H'], 'W': c['W'],
                  'frames': c['frames_per_gpu'], 'Gpx_s': d['value']/1e3, 'fps': c['fps'], 'frac': d['roofline']['frac'],
                  'variant': c['kernel_variant'], 'clocks': d['clocks']}))"
}
for f in fd scharr; do for m in mean median; do run --config 3 --filter $f --mode $m; done; done
run --config 4
run --config 4 --hw 2160,3840 --frames 32
run --config 4 --hw 2160,3840 --frames 32 --holes 0
