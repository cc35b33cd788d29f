timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
rm -f gpurun_out/tune.jsonl
run() { local envs=$1; shift; local out; out=$(env $envs timeout 300 python bench.py --no-cpu --steps 50 --warmup 5 "$@" 2>>gpurun_out/tune_err.log | tail -1); [ -n "$out" ] && python -c "import json,sys; d=json.loads(sys.argv[1]); d['env']=sys.argv[2]; print(json.dumps(d))" "$out" "$envs" >> gpurun_out/tune.jsonl; }
for cfg in c2 pent512 tri512; do
  for mode in exact fast; do
    for w in 2 3 4; do run "BANDSOLVE_PWARPS=$w" --config $cfg --mode $mode; done
  done
done
BANDSOLVE_PWARPS=4 bash tools/gpu_ncu.sh pent512_exact_rr --config pent512 --mode exact
