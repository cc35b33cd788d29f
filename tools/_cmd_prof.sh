cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in "c4tri" "c4pent"; do
BANDSOLVE_PART_K=16 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launch_$c.csv python bench.py --no-cpu --config $c --mode fast --steps 2 --warmup 1 > /dev/null 2>&1
done
