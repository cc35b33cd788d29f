#!/bin/bash
# Plan-knob sweep: KNOB_SPECS="cfg:mode:ENV=V,ENV2=V ..." -> gpurun_out/knobs.jsonl
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/${KNOB_OUT:-knobs}.jsonl
rm -f $out
for spec in $KNOB_SPECS; do
  IFS=: read -r cfg mode envs <<< "$spec"
  r=$(env ${envs//,/ } timeout 180 python bench.py --no-cpu --steps ${STEPS:-20} --warmup 3 --config $cfg --mode $mode ${BENCH_EXTRA:-} 2>>gpurun_out/knobs_err.log | tail -n 1)
  [ -n "$r" ] && python -c "import json,sys; d=json.loads(sys.argv[1]); d['env']=sys.argv[2]; print(json.dumps(d))" "$r" "$envs" >> $out
done
python - "$out" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); c=d['config']
    print(f"{c['kind']:5s} {c['n']:5d} {c['batch_per_gpu']:8d} {c['mode']:6s} {d['env'][:34]:34s} {d['value']:.3e} frac={d['roofline']['frac']:.3f} {c['plan'][:80]}")
PY
