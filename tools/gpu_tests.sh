#!/bin/bash
# GPU test suite + smoke + default bench at HEAD (output under gpurun_out/).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1; free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
for i in ${RUNS:-1}; do
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$i.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_err.log
tail -3 gpurun_out/pytest_gpu_*.log; cat gpurun_out/smoke.log gpurun_out/bench_default.json
