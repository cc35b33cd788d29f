#!/bin/bash
# Round artifacts on one B200: GPU tests, smoke, bench lines (default, reference
# arm, config sweep), ncu launch list + full captures. Output under gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
if [ -z "${SKIP_TESTS:-}" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
timeout 600 python bench.py > gpurun_out/bench_default.json 2>> gpurun_out/bench_err.log
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench_err.log
rm -f gpurun_out/bench_sweep.jsonl
for mode in exact fast; do
  for cfg in c1 c2 tri512 pent512 c5; do
    timeout 300 python bench.py --config $cfg --mode $mode --no-cpu --steps 50 --warmup 5 >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_err.log
  done
done
timeout 300 python bench.py --config tri512 --f32 --no-cpu --steps 50 --warmup 5 >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_err.log
for extra in "--config pent512 --periodic" "--config pent512 --periodic --mode fast" "--config pent512 --cn" "--config pent512 --cn --mode fast" "--config tri512 --cn --mode fast" "--config c4tri" "--config c4tri --mode fast" "--config c4pent" "--config c4pent --mode fast"; do
  timeout 300 python bench.py $extra --no-cpu --steps 20 --warmup 3 >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_err.log
done
timeout 300 python bench.py --config pent512 --f32 --no-cpu --steps 50 --warmup 5 >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_err.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
   --log-file gpurun_out/launches_c4tri_fast.csv python bench.py --config c4tri --mode fast --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
for cfg in ${NCU_CFGS:-c2}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_ -s 3 -c 1 \
    -o gpurun_out/prof_r1_${cfg} -f python bench.py --config $cfg --no-cpu --steps 3 --warmup 3 > gpurun_out/ncu_${cfg}.log 2>&1
done
du -sh gpurun_out/*; cat gpurun_out/bench_default.json gpurun_out/bench_ref.json
