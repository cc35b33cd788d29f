#!/bin/bash
# GPU tests + stream-plan sweep. Output under gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
rm -f gpurun_out/tune.jsonl
run() { local envs=$1; shift; local out; out=$(env $envs timeout 120 python bench.py --no-cpu --steps 30 --warmup 5 "$@" 2>>gpurun_out/tune_err.log | tail -1); [ -n "$out" ] && python -c "import json,sys; d=json.loads(sys.argv[1]); d['env']=sys.argv[2]; print(json.dumps(d))" "$out" "$envs" >> gpurun_out/tune.jsonl; }
for cfg in c2 pent512 tri512 c5 c1; do
  for mode in exact fast; do
    run "BANDSOLVE_X=0" --config $cfg --mode $mode
  done
done
for cfg in pent512 tri512 c2; do
 for mode in exact fast; do
 for wg in 64 128 192; do
  for kr in 3 4; do
      run "BANDSOLVE_SWG=$wg BANDSOLVE_SKR=$kr" --config $cfg --mode $mode
  done
 done
 done
done
for wg in 64 128; do
  run "BANDSOLVE_SWG=$wg" --config tri512 --mode exact --n 256 --m 2097152
  run "BANDSOLVE_SWG=$wg" --config pent512 --mode exact --n 256 --m 2097152
done
python - <<'PY'
import json
for l in open('gpurun_out/tune.jsonl'):
    d=json.loads(l); c=d['config']
    print(f"{c['kind']:5s} {c['n']:5d} {c['batch_per_gpu']:8d} {c['mode']:6s} {d['env'][:40]:40s} {d['value']:.3e} frac={d['roofline']['frac']:.3f} {c['plan'][:72]}")
PY
