#!/bin/bash
# GPU tests + targeted bench lines listed as "ENV|ARGS" entries (one per line) in tools/quick_runs.txt.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
[ -z "${SKIP_TESTS:-}" ] && timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/quick.jsonl
while IFS='|' read -r envs args; do
  [ -z "$args" ] && continue
  out=$(env $envs timeout 120 python bench.py --no-cpu --steps 30 --warmup 5 $args 2>>gpurun_out/tune_err.log | tail -1)
  [ -n "$out" ] && python -c "import json,sys; d=json.loads(sys.argv[1]); d['env']=sys.argv[2]; print(json.dumps(d))" "$out" "$envs" >> gpurun_out/quick.jsonl
done < tools/quick_runs.txt
python - <<'PY'
import json
for l in open('gpurun_out/quick.jsonl'):
    d=json.loads(l); c=d['config']
    e=d.get('e2e') or {}
    print(f"{c['kind']:5s} {c['n']:5d} {c['batch_per_gpu']:8d} {c['mode']:6s} {d['env'][:40]:40s} {d['value']:.3e} frac={d['roofline']['frac']:.3f} e2e={e.get('value',0):.3e} {c['plan'][:60]}")
PY
