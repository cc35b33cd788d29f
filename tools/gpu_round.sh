#!/bin/bash
# One gpurun session: GPU tests, smoke, bench lines. Output under gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for mode in exact fast; do
  for cfg in c2 c1 tri512 pent512; do
    timeout 300 python bench.py --config $cfg --mode $mode --no-cpu --steps 100 --warmup 10 >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_err.log
  done
done
timeout 600 python bench.py > gpurun_out/bench_default.json 2>> gpurun_out/bench_err.log
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; cat gpurun_out/bench_default.json
