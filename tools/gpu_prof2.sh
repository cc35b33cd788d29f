#!/bin/bash
# Round-2 profiling: ncu full captures (with source) of the stream sweep at the
# north-star shape and the configs[4] shard, plus a small plan sweep.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for spec in "pent512 exact" "c5 exact" "c5 fast"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_ -s 2 -c 1 \
    -o gpurun_out/prof_r2_$1_$2 -f python bench.py --config $1 --mode $2 --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu_$1_$2.log 2>&1
done
rm -f gpurun_out/tune.jsonl
run() { local envs=$1; shift; local out; out=$(env $envs timeout 120 python bench.py --no-cpu --steps 20 --warmup 3 "$@" 2>>gpurun_out/tune_err.log | tail -n 1); [ -n "$out" ] && python -c "import json,sys; d=json.loads(sys.argv[1]); d['env']=sys.argv[2]; print(json.dumps(d))" "$out" "$envs" >> gpurun_out/tune.jsonl; }
for mode in exact fast; do
  for e in "X=0" "BANDSOLVE_SWG=64" "BANDSOLVE_SWG=96" "BANDSOLVE_SWG=128" "BANDSOLVE_TMEM=0" "BANDSOLVE_PLAN=global"; do
    run "$e" --config c5 --mode $mode
  done
  for e in "X=0" "BANDSOLVE_SWG=96" "BANDSOLVE_SWG=64" "BANDSOLVE_SKB=6" "BANDSOLVE_SKR=6" "BANDSOLVE_SPD=8"; do
    run "$e" --config pent512 --mode $mode
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/tune.jsonl'):
    d=json.loads(l); c=d['config']
    print(f"{c['kind']:5s} {c['n']:5d} {c['batch_per_gpu']:8d} {c['mode']:6s} {d['env'][:30]:30s} {d['value']:.3e} frac={d['roofline']['frac']:.3f} {c['plan'][:90]}")
PY
