mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bag or layer" > gpurun_out/pytest_pipe.log 2>&1; echo pytest_exit=$?
tail -1 gpurun_out/pytest_pipe.log
ML_SEG_PIPE_CFG=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bag or layer" > gpurun_out/pytest_pipe1.log 2>&1; echo pytest_cfg1_exit=$?
tail -1 gpurun_out/pytest_pipe1.log
for cfg in ${CFGS:-2 1}; do
ML_SEG_PIPE_CFG=$cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$cfg.log 2>&1; echo bench_$cfg exit=$?
MODE="$cfg" python - <<'PY'
import json, os
f = 'gpurun_out/bench_cfg%s.log' % os.environ["MODE"]
l = [x for x in open(f) if x.startswith('{')]
if l:
    d = json.loads(l[-1]); print(os.environ["MODE"], "value", d["value"], "ms", d["ms_per_step"]); k = d["kernel_ms_per_step"]; print({x: k[x] for x in list(k)[:5]})
else:
    print(open(f).read()[-3000:])
PY
done
