#!/bin/bash
# GPU tests + stream-plan calibration sweep -> gpurun_out/calib.jsonl
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/calib.jsonl
run() { local envs=$1; shift; local out; out=$(env $envs timeout 120 python bench.py --no-cpu --steps 15 --warmup 3 "$@" 2>>gpurun_out/tune_err.log | tail -1); [ -n "$out" ] && python -c "import json,sys; d=json.loads(sys.argv[1]); d['env']=sys.argv[2]; print(json.dumps(d))" "$out" "$envs" >> gpurun_out/calib.jsonl; }
for shape in "256 2097152" "512 1048576" "1024 524288"; do
 set -- $shape; n=$1; m=$2
 for cfg in tri512 pent512; do
  for mode in exact fast; do
   for vw in "1 64" "1 96" "1 128" "1 160" "2 64" "2 128" "2 192"; do
     set -- $vw
     run "BANDSOLVE_SV=$1 BANDSOLVE_SWG=$2 BANDSOLVE_SKR=4" --config $cfg --mode $mode --n $n --m $m
   done
  done
 done
done
python - <<'PY'
import json
for l in open('gpurun_out/calib.jsonl'):
    d=json.loads(l); c=d['config']
    print(f"{c['kind']:5s} {c['n']:5d} {c['mode']:6s} {d['env'][:44]:44s} frac={d['roofline']['frac']:.3f} {c['plan'][7:60]}")
PY
