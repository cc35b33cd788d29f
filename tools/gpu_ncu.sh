#!/bin/bash
# ncu capture of the sweep kernel (one GPU). Usage: tools/gpu_ncu.sh <tag> <bench args...>
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
tag=$1; shift
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_ -s 3 -c 1 \
    -o gpurun_out/prof_${tag} -f python bench.py --no-cpu --steps 3 --warmup 3 "$@" > gpurun_out/ncu_${tag}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_${tag}.log
