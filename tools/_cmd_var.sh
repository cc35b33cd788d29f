cd $GRAFT_REPO_ROOT
run() { python bench.py --no-cpu --steps 20 --warmup 3 "$@" | python -c "import json,sys,os; d=json.loads(sys.stdin.read()); c=d['config']; print(c['kind'], c['mode'], os.environ.get('BANDSOLVE_PART_K'), '%.3e'%d['value'], '%.3f ms'%d['ms_per_step'])" "$@"; }
for r in 1 2; do run --config c4pent --mode fast; done
for r in 1 2; do run --config c4tri --mode fast; done
BANDSOLVE_PART_K=16 run --config c4pent --mode fast
BANDSOLVE_PART_K=16 run --config c4tri --mode fast
timeout 600 python -m pytest tests/test_partition.py tests/test_adi.py -q -x 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c4tri_fast.csv python bench.py --config c4tri --mode fast --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
