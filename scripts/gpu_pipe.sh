mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bag or layer" > gpurun_out/pytest_pipe.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|FAILED|Error|error" gpurun_out/pytest_pipe.log | tail -8
for cfg in ${CFGS:-"1 256 64" "1 128 64" "1 256 12" "0 256 64"}; do
set -- $cfg
ML_SEG_PIPE=$1 ML_SEG_TEAM=$2 ML_SEG_SLOTS=$3 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pipe$1_$2_$3.log 2>&1; echo bench_$1_$2_$3 exit=$?
MODE="$1_$2_$3" python - <<'PY'
import json, os
f = 'gpurun_out/bench_pipe%s.log' % os.environ["MODE"]
l = [x for x in open(f) if x.startswith('{')]
if l:
    d = json.loads(l[-1]); print(os.environ["MODE"], "value", d["value"], "ms", d["ms_per_step"]); k = d["kernel_ms_per_step"]; print({x: k[x] for x in list(k)[:5]})
else:
    print(open(f).read()[-3000:])
PY
done
