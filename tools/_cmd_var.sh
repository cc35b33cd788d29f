cd $GRAFT_REPO_ROOT
run() { python bench.py --no-cpu --steps 10 --warmup 3 "$@" | python -c "import json,sys,os; d=json.loads(sys.stdin.read()); c=d['config']; print(c['kind'], c['n'], c['batch_per_gpu'], d['dtype'], c['mode'], os.environ.get('BANDSOLVE_PLAN'), '%.3e'%d['value'], 'frac=%.3f'%d['roofline']['frac'], c['plan'][:30])" "$@"; }
for m in 16384 65536 262144; do
  run --config tri512 --n 2048 --m $m
  BANDSOLVE_PLAN=global run --config tri512 --n 2048 --m $m
done
run --config tri512 --n 1536 --m 1048576
BANDSOLVE_PLAN=global run --config tri512 --n 1536 --m 1048576
BANDSOLVE_PLAN=global run --config tri512 --n 2048 --m 1048576 --f32
BANDSOLVE_PLAN=global run --config tri512 --n 4096 --m 1048576 --f32
BANDSOLVE_PLAN=global run --config tri512 --n 1024 --m 1048576 --f32
BANDSOLVE_PLAN=global run --config tri512 --n 2048 --m 1048576 --mode fast
