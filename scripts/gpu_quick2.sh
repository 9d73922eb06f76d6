mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo bench_exit=$?
python - <<'PY'
import json
l = [x for x in open('gpurun_out/bench_q.log') if x.startswith('{')]
if l:
    d = json.loads(l[-1]); print("value", d["value"], "ms", d["ms_per_step"]); k = d["kernel_ms_per_step"]; print(k)
else:
    print(open('gpurun_out/bench_q.log').read()[-3000:])
PY
