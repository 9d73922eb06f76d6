mkdir -p gpurun_out
timeout 900 python bench.py ${BENCH_ARGS:---cpu-tokens 256} > gpurun_out/bench.log 2>gpurun_out/bench.err; echo bench_exit=$?
python - <<'PY'
import json
l = [x for x in open('gpurun_out/bench.log') if x.startswith('{')]
if l:
    d = json.loads(l[-1]); print("value", d["value"], "ms", d["ms_per_step"]); print("e2e", d["e2e"]); print(d["roofline"]); print(d["kernel_ms_per_step"]); print(d["clocks"], d["gpu_launches"])
else:
    print(open('gpurun_out/bench.err').read()[-3000:])
PY
