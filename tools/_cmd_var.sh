cd $GRAFT_REPO_ROOT
run() { python bench.py --no-cpu --steps 20 --warmup 3 "$@" | python -c "import json,sys,os; d=json.loads(sys.stdin.read()); c=d['config']; print(c['kind'], c['mode'], os.environ.get('BANDSOLVE_PART_K'), '%.3e'%d['value'], '%.3f ms'%d['ms_per_step'], d['gpu_launches'])" "$@"; }
timeout 600 python -m pytest tests/test_adi.py -q -x 2>&1 | tail -1
run --config c4tri --mode fast
run --config c4tri --mode fast
BANDSOLVE_PART_K=8 run --config c4tri --mode fast
