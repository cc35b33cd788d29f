#!/bin/bash
# Tuning-key A/B on one box: ENV_SPECS="cfg:mode:KEY=V,KEY2=V[:--n+768] ..."
# (BANDSOLVE_ prefix added; "-" = defaults; '+' in the optional 4th field =
# space, extra bench.py args) -> gpurun_out/env.txt
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/env.txt; : > $out
for spec in ${ENV_SPECS}; do
  IFS=: read -r cfg mode envs xargs <<< "$spec"
  e=(); [ "$envs" != "-" ] && for kv in ${envs//,/ }; do e+=("BANDSOLVE_$kv"); done
  r=$(env "${e[@]}" X=1 timeout 240 python bench.py --config $cfg --mode $mode --no-cpu --no-e2e ${ENV_ARGS:-} ${xargs//+/ } --steps ${ENV_STEPS:-20} --warmup 5 2>gpurun_out/env_err.txt | tail -1)
  python - "$r" "$spec" >> $out <<'PY'
import json,sys
r=json.loads(sys.argv[1]) if sys.argv[1].startswith('{') else {}
print(f'{sys.argv[2]:50s}', round(r.get("roofline",{}).get("frac",0) or 0,4), r.get("config",{}).get("plan","")[:110])
PY
done
cat $out
