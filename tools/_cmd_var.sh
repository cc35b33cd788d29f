cd $GRAFT_REPO_ROOT
run() { python bench.py --no-cpu --steps 50 --warmup 5 "$@" | python -c "import json,sys,os; d=json.loads(sys.stdin.read()); c=d['config']; print(c['kind'], c['n'], c['batch_per_gpu'], c['mode'], os.environ.get('BANDSOLVE_SPLIT'), '%.3e'%d['value'], 'frac=%.3f'%d['roofline']['frac'], d['gpu_launches'])" "$@"; }
BANDSOLVE_SPLIT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "config2 or config1 or pent_n512" 2>&1 | tail -1
run --config c2
BANDSOLVE_SPLIT=1 run --config c2
run --config c2 --mode fast
BANDSOLVE_SPLIT=1 run --config c2 --mode fast
run --config pent512
BANDSOLVE_SPLIT=1 run --config pent512
run --config tri512
BANDSOLVE_SPLIT=1 run --config tri512
