#!/bin/bash
# ncu --set full captures (with source) for the given "config mode [env]" specs;
# reports stay on the box (/tmp), only CSV exports come back under gpurun_out/.
# Usage: NCU_SPECS="pent512:exact c5s:exact" bash tools/gpu_ncu.sh
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/ncu /tmp/ncurep
for spec in ${NCU_SPECS:-pent512:exact}; do
  IFS=: read -r cfg mode envs <<< "$spec"
  tag="${cfg}_${mode}${envs:+_$(echo $envs | tr '=,' '__')}"
  env ${envs//,/ } timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KREGEX:-sweep_} -s ${NCU_SKIP:-2} -c 1 \
    -o /tmp/ncurep/$tag -f python bench.py --config $cfg --mode $mode --no-cpu --steps 2 --warmup 3 ${BENCH_EXTRA:-} > gpurun_out/ncu/$tag.log 2>&1
  ncu -i /tmp/ncurep/$tag.ncu-rep --page raw --csv > gpurun_out/ncu/$tag.raw.csv 2>>gpurun_out/ncu/$tag.log
  ncu -i /tmp/ncurep/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/$tag.sass.csv 2>>gpurun_out/ncu/$tag.log
  gzip -f gpurun_out/ncu/$tag.sass.csv
done
du -sh gpurun_out/ncu/*
