mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_large_s.py tests/test_gpu_parity.py -k "pkm or fused or layer" -q -x -p no:cacheprovider -rf > gpurun_out/r2g_pytest.log 2>&1; echo exit=$?; grep -E "passed|failed|Error|error" gpurun_out/r2g_pytest.log | head -10
for cfg in "--config c2" "--config c4 --per-rank 8"; do
timeout 300 python bench.py $cfg --steps 10 --no-cpu-baseline --no-variants > gpurun_out/r2g_bench.log 2>&1; python -c "
import json
d=json.loads([x for x in open('gpurun_out/r2g_bench.log') if x.startswith('{')][-1])
print(d['ms_per_step']); print(d['kernel_ms_per_step']); print(d['scoring_roofline'])
"; done
