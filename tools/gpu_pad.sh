#!/bin/bash
# Row-pitch (partition camping) probe: configs[4] at 2^24 with padded pitches.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for spec in ${PAD_SPECS:-"fast 0" "fast 32" "fast 64" "fast 256" "fast 1024" "exact 0" "exact 64"}; do
  set -- $spec
  timeout 300 python bench.py --config ${PAD_CFG:-c5} --mode $1 --pitch-pad $2 --no-cpu --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 pad=$2', round(d['roofline']['frac'],4), d['ms_per_step'])"
done
