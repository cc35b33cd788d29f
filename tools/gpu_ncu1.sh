#!/bin/bash
# One ncu --set full capture: tools/gpu_ncu1.sh <cfg> <mode> <kernel regex> [tag] [bench args...]
# -> gpurun_out/ncu/<tag>.{raw.csv,details.csv,sass.csv.gz,log}
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/ncu /tmp/ncurep
cfg=$1 mode=$2 kre=$3; tag=${4:-${cfg}_${mode}}; shift 4 2>/dev/null || shift $#
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 3 -c 1 \
  -o /tmp/ncurep/$tag -f python bench.py --config $cfg --mode $mode --no-cpu --no-e2e --steps 2 --warmup 3 "$@" > gpurun_out/ncu/$tag.log 2>&1
ncu -i /tmp/ncurep/$tag.ncu-rep --page raw --csv > gpurun_out/ncu/$tag.raw.csv 2>>gpurun_out/ncu/$tag.log
ncu -i /tmp/ncurep/$tag.ncu-rep --page details --csv > gpurun_out/ncu/$tag.details.csv 2>>gpurun_out/ncu/$tag.log
ncu -i /tmp/ncurep/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/$tag.sass.csv 2>>gpurun_out/ncu/$tag.log
gzip -f gpurun_out/ncu/$tag.sass.csv
