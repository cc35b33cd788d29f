#!/bin/bash
# Bench sweep over plan overrides. Appends JSON lines (with an "env" key) to gpurun_out/tune.jsonl.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
run() {  # run "<env assignments>" <bench args...>
  local envs=$1; shift
  local out
  out=$(env $envs timeout 300 python bench.py --no-cpu --steps 50 --warmup 5 "$@" 2>>gpurun_out/tune_err.log | tail -1)
  [ -n "$out" ] && python -c "import json,sys; d=json.loads(sys.argv[1]); d['env']=sys.argv[2]; print(json.dumps(d))" "$out" "$envs" >> gpurun_out/tune.jsonl
}
for cfg in c2 tri512 pent512; do
  for mode in exact fast; do
    run "X=1" --config $cfg --mode $mode
    for w in 2 3 4 6; do run "BANDSOLVE_PWARPS=$w" --config $cfg --mode $mode; done
  done
done
run "X=1" --config c1
run "BANDSOLVE_PLAN=smemW16" --config c2
