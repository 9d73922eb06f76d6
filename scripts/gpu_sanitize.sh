mkdir -p gpurun_out
# memcheck on the small parity cases (one sanitizer tool per call)
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "not 2048 and not 4096 and not 1024-1024" > gpurun_out/sanitize_memcheck.log 2>&1; echo memcheck_exit=$?
grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_memcheck.log | tail -5
