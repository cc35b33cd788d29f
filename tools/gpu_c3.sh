#!/bin/bash
# configs[2]: tri N in {64..4096}, 2^20 systems, fp64 exact/fast and fp32.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f gpurun_out/c3_sweep.jsonl
for n in 64 128 256 512 1024 2048 4096; do
  for extra in "" "--mode fast" "--f32"; do
    timeout 300 python bench.py --config tri512 --n $n --m 1048576 $extra --no-cpu --steps 10 --warmup 3 >> gpurun_out/c3_sweep.jsonl 2>> gpurun_out/c3_err.log
  done
done
wc -l gpurun_out/c3_sweep.jsonl
