#!/bin/bash
# A/B of library builds on one box: AB_DIRS="dirA dirB ..." (repo copies with
# their own built .so; "." = this tree), AB_SPECS="cfg:mode ..." -> gpurun_out/ab.jsonl
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/ab.jsonl; rm -f $out
for rep in ${AB_REPS:-1 2}; do
for spec in ${AB_SPECS:-pent512:exact tri512:exact c2:exact pent512:fast}; do
  IFS=: read -r cfg mode <<< "$spec"
  for d in ${AB_DIRS:-.}; do
    extra=""; [ -f "$d/bench.py" ] && grep -q no-e2e "$d/bench.py" && extra="--no-e2e"
    r=$(cd $d && timeout 180 python bench.py --config $cfg --mode $mode --no-cpu $extra --steps ${AB_STEPS:-30} --warmup 5 2>/dev/null | tail -1)
    python - "$r" "$d" "$spec" >> $out <<'PY'
import json,sys
r=json.loads(sys.argv[1]) if sys.argv[1].startswith('{') else {}
print(json.dumps({"spec":sys.argv[3],"dir":sys.argv[2],"frac":r.get("roofline",{}).get("frac"),"plan":r.get("config",{}).get("plan","")[:90]}))
PY
  done
done
done
python - $out <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(f"{d['spec']:16s} {d['dir']:8s} {d['frac'] if d['frac'] is None else round(d['frac'],4)}  {d['plan']}")
PY
