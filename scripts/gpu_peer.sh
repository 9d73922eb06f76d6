mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -x > gpurun_out/pytest_peer.log 2>&1; echo peer_exit=$?
grep -E "passed|failed|Error|assert|FAILED" gpurun_out/pytest_peer.log | tail -15
