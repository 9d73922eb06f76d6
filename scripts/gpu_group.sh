mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_group.py -q -p no:cacheprovider -x > gpurun_out/pytest_group.log 2>&1; echo group_exit=$?
tail -25 gpurun_out/pytest_group.log
