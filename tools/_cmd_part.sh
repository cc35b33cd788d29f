cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_partition.py tests/test_periodic.py tests/test_adi.py tests/test_gpu_parity.py -k "partition or fast or adi" -x -q > gpurun_out/pytest_part.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_part.log; tail -15 gpurun_out/pytest_part.log
SKIP_TESTS=1 bash tools/gpu_quick.sh
