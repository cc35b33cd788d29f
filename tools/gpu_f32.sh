#!/bin/bash
# fp32 spike sweep: N x kind, fast mode -> gpurun_out/f32.txt
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/f32.txt; : > $out
for kind in tri pent; do
for n in ${F32_NS:-256 512 1024 2048 4096}; do
  for env in ${F32_ENVS:-none}; do
    r=$(env ${env/none/X=1} timeout 180 python bench.py --config ${kind}512 --n $n --m ${F32_M:-1048576} --f32 --mode fast --no-cpu --no-e2e --steps 20 --warmup 5 2>/dev/null | tail -1)
    python - "$r" "$kind $n $env" >> $out <<'PY'
import json,sys
r=json.loads(sys.argv[1]) if sys.argv[1].startswith('{') else {}
print(sys.argv[2], round(r.get("roofline",{}).get("frac",0) or 0,4), r.get("config",{}).get("plan","")[:80])
PY
  done
done
done
cat $out
