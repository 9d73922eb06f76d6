mkdir -p gpurun_out
ML_SEG_TEAM=64 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bag or layer" > gpurun_out/pytest_team64.log 2>&1; echo pytest64_exit=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_team64.log | tail -5
for team in 256 128 64 32; do
ML_SEG_TEAM=$team timeout 600 python bench.py --steps 10 --warmup 3 --cpu-tokens 64 > gpurun_out/bench_team$team.log 2>&1; echo bench_$team exit=$?
MODE=$team python - <<'PY'
import json, os
l = [x for x in open('gpurun_out/bench_team%s.log' % os.environ["MODE"]) if x.startswith('{')]
if l:
    d = json.loads(l[-1]); print(os.environ["MODE"], "value", d["value"], "ms", d["ms_per_step"]); k = d["kernel_ms_per_step"]; print({x: k[x] for x in list(k)[:6]})
else:
    print(open('gpurun_out/bench_team%s.log' % os.environ["MODE"]).read()[-3000:])
PY
done
