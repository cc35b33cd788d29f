#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family
# (tools/sanitize/drive.py). Logs under gpurun_out/sanitize/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${SAN_TOOLS:-memcheck synccheck racecheck}; do
  for fam in ${SAN_FAMS:-stream other_plans spike spike_variants pipe partition periodic cn_adi host per_system}; do
    timeout ${SAN_TIMEOUT:-900} $CS --tool $tool --target-processes all --print-limit 20 --error-exitcode 77 \
      python tools/sanitize/drive.py $fam > gpurun_out/sanitize/${tool}_${fam}.log 2>&1
    echo "$tool $fam rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|DRIVE OK' gpurun_out/sanitize/${tool}_${fam}.log | tr '\n' ' ')"
  done
done | tee gpurun_out/sanitize/summary.txt
# racecheck on the minimal mbarrier ring (1D bulk copy vs 2D tensor load):
# tells a tool report on the reload-ring protocol from a real race
( cd tools/sanitize && nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o bulk_ring bulk_ring.cu -lcuda &&
  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -DTENSOR -o tensor_ring bulk_ring.cu -lcuda ) > /dev/null 2>&1
for b in bulk_ring tensor_ring; do
  $CS --tool racecheck tools/sanitize/$b > gpurun_out/sanitize/racecheck_repro_$b.log 2>&1
  echo "racecheck repro $b: $(grep -E 'ring:|RACECHECK SUMMARY' gpurun_out/sanitize/racecheck_repro_$b.log | tr '\n' ' ')"
done | tee -a gpurun_out/sanitize/summary.txt
# racecheck on the cluster interface exchange (mbarrier vs barrier.cluster)
( cd tools/sanitize && nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o cluster_xch cluster_xch.cu &&
  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -DHWBAR -o cluster_xch_hw cluster_xch.cu ) > /dev/null 2>&1
for b in cluster_xch cluster_xch_hw; do
  $CS --tool racecheck tools/sanitize/$b > gpurun_out/sanitize/racecheck_repro_$b.log 2>&1
  echo "racecheck repro $b: $(grep -E 'exchange:|RACECHECK SUMMARY' gpurun_out/sanitize/racecheck_repro_$b.log | tr '\n' ' ')"
done | tee -a gpurun_out/sanitize/summary.txt
