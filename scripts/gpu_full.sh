mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > gpurun_out/pytest_full.log 2>&1; echo full_exit=$?
tail -30 gpurun_out/pytest_full.log
