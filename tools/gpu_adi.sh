#!/bin/bash
# Few-system regimes (configs[0], configs[3] ADI): per-launch breakdown of one
# bench step (ncu launch list), fp64 dependent-op latency, PCIe copy rates.
# Output under gpurun_out/adi/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/adi
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dplat tools/microbench/dplat.cu > $O/dplat.log 2>&1 && /tmp/dplat >> $O/dplat.log 2>&1
timeout 120 python tools/pcie_bw.py > $O/pcie.log 2>&1
for spec in "c4tri exact" "c4pent exact" "c4tri fast" "c4pent fast" "c1 exact" "c1 fast"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --mode $2 --no-cpu --no-e2e --steps 20 --warmup 3 >> $O/bench.jsonl 2>> $O/err.log
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv \
     --log-file $O/launch_${1}_${2}.csv python bench.py --config $1 --mode $2 --no-cpu --no-e2e --steps 1 --warmup 3 > /dev/null 2>> $O/err.log
done
cat $O/dplat.log $O/pcie.log $O/bench.jsonl | cut -c1-400
