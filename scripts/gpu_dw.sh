mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -12
for mode in token fused; do
ML_BAG_DW=$mode timeout 600 python bench.py --steps 10 --warmup 3 --cpu-tokens 64 > gpurun_out/bench_$mode.log 2>&1; echo bench_$mode exit=$?
MODE=$mode python - <<'PY'
import json, os
l = [x for x in open('gpurun_out/bench_%s.log' % os.environ["MODE"]) if x.startswith('{')]
if l:
    d = json.loads(l[-1]); print(os.environ["MODE"], "value", d["value"], "ms", d["ms_per_step"]); print(d["roofline"]); print(d["kernel_ms_per_step"])
else:
    print(open('gpurun_out/bench_%s.log' % os.environ["MODE"]).read()[-3000:])
PY
done
