#!/bin/bash
# A/B: the round-1 library (worktree _ab_r1, built there) vs HEAD on the same box.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/ab.jsonl; rm -f $out
for rep in 1 2; do
for spec in "pent512 exact" "tri512 exact" "c2 exact" "pent512 fast"; do
  set -- $spec
  a=$(cd _ab_r1 && timeout 120 python bench.py --config $1 --mode $2 --no-cpu --steps 30 --warmup 5 2>/dev/null | tail -1)
  b=$(timeout 120 python bench.py --config $1 --mode $2 --no-cpu --no-e2e --steps 30 --warmup 5 2>/dev/null | tail -1)
  python - "$a" "$b" "$1 $2" >> $out <<'PY'
import json,sys
a=json.loads(sys.argv[1]) if sys.argv[1] else {}
b=json.loads(sys.argv[2]) if sys.argv[2] else {}
print(json.dumps({"spec":sys.argv[3],"r1":a.get("roofline",{}).get("frac"),"head":b.get("roofline",{}).get("frac")}))
PY
done
done
cat $out
