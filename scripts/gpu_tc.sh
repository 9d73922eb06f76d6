mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "pkm" -x > gpurun_out/pytest_pkm.log 2>&1; echo pkm_exit=$?
grep -E "passed|failed|FAILED|Error|error" gpurun_out/pytest_pkm.log | tail -12
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | tail -12
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-tokens 64 > gpurun_out/bench.log 2>&1; echo bench_exit=$?
python - <<'PY'
import json
l = [x for x in open('gpurun_out/bench.log') if x.startswith('{')]
if l:
    d = json.loads(l[-1]); print("value", d["value"], "ms", d["ms_per_step"]); print(d["roofline"]); print(d["bag_kernels"]); print(d["kernel_ms_per_step"])
else:
    print(open('gpurun_out/bench.log').read()[-3000:])
PY
