#!/bin/bash
# Round-2 artifacts on one B200: GPU tests, smoke, default bench + reference
# arm, a config sweep (exact and fast), ncu launch list of the default bench
# and ncu --set full captures (raw + source CSV exports) of the hot kernels.
# Output under gpurun_out/ (SKIP_TESTS=1 / SKIP_SWEEP=1 / SKIP_NCU=1 to skip parts).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/ncu /tmp/ncurep
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_err.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench_err.log
if [ -z "${SKIP_SWEEP:-}" ]; then
  rm -f gpurun_out/bench_sweep.jsonl
  for mode in fast exact; do
    for cfg in c1 c2 tri512 pent512 c5s c5; do
      st=30; [ $cfg = c5 ] && st=5
      timeout 300 python bench.py --config $cfg --mode $mode --no-cpu --no-e2e --steps $st --warmup 3 >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_err.log
    done
    for nn in 64 128 256 1024 2048 4096; do  # configs[2]: tri, 2^20 systems, N sweep
      timeout 300 python bench.py --config tri512 --n $nn --m 1048576 --mode $mode --no-cpu --no-e2e --steps 10 --warmup 3 >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_err.log
      timeout 300 python bench.py --config tri512 --n $nn --m 1048576 --f32 --mode $mode --no-cpu --no-e2e --steps 10 --warmup 3 >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_err.log
    done
    timeout 300 python bench.py --config tri512 --f32 --mode $mode --no-cpu --steps 30 --warmup 3 >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_err.log
    for extra in "--config pent512 --periodic" "--config tri512 --periodic" "--config pent512 --cn" "--config tri512 --cn" "--config c4tri" "--config c4pent"; do
      timeout 300 python bench.py $extra --mode $mode --no-cpu --no-e2e --steps 20 --warmup 3 >> gpurun_out/bench_sweep.jsonl 2>> gpurun_out/bench_err.log
    done
  done
fi
if [ -z "${SKIP_NCU:-}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
     --log-file gpurun_out/launches_default.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
  for spec in "c5s fast sweep_spike" "pent512 fast sweep_spike" "tri512 fast sweep_spike" "pent512 exact sweep_pipe" \
              "c2 exact sweep_pipe" "c2 fast sweep_spike" "c5s exact sweep_pipe" "tri512 fast sweep_spike tri512f32_fast --f32"; do
    set -- $spec
    bash tools/gpu_ncu1.sh "$@"
  done
fi
tail -3 gpurun_out/pytest_gpu.log 2>/dev/null; cat gpurun_out/smoke.log 2>/dev/null; cat gpurun_out/bench_default.json gpurun_out/bench_ref.json
