#!/bin/bash
# A/B with a correctness gate: smoke (parity vs the oracle + general-variant bit identity)
# per library, then tools/ab.sh throughput.  Usage: tools/ab_check.sh libA.so libB.so ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for lib in "$@"; do
  TFN_LIB=$lib timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$(basename $lib).log 2>&1
  echo "$lib smoke_rc=$?"
done
bash tools/ab.sh "$@"
