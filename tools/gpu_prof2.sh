#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
prof() { local tag=$1; shift; timeout 300 env "$@" ncu --set full --clock-control none --import-source on -k regex:sweep_ -s 3 -c 1 -o gpurun_out/prof_$tag -f python bench.py --no-cpu --steps 3 --warmup 3 $BENCH_ARGS > gpurun_out/ncu_$tag.log 2>&1; echo "$tag rc=$?"; }
BENCH_ARGS="--config pent512 --mode fast" prof v6_pent512f_64 BANDSOLVE_SWG=64 BANDSOLVE_SV=1 BANDSOLVE_SKR=4
