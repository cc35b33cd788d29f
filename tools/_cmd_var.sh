cd $GRAFT_REPO_ROOT
run() { python bench.py --no-cpu --steps 20 --warmup 3 "$@" | python -c "import json,sys,os; d=json.loads(sys.stdin.read()); c=d['config']; print(c['kind'], c['mode'], os.environ.get('BANDSOLVE_PART_K'), '%.3e'%d['value'], '%.3f ms'%d['ms_per_step'])" "$@"; }
for r in 1 2 3 4 5; do run --config c4pent --mode fast; done
for r in 1 2 3 4 5; do run --config c4tri --mode fast; done
