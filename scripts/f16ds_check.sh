# fp16 operands of the tcgen05 key backward: parity + C2 A/B against the bf16 path
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pkm_bwd_split.py -q -p no:cacheprovider -s -x > gpurun_out/f16_pytest.log 2>&1; echo split_exit=$?; grep -E "max rel|passed|failed|Error" gpurun_out/f16_pytest.log | tail -8
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layer_autograd.py tests/test_gpu_large_s.py -q -p no:cacheprovider -x -k "bwd or layer or deterministic" > gpurun_out/f16_parity.log 2>&1; echo parity_exit=$?; tail -1 gpurun_out/f16_parity.log
for c in 1 0 1 0 1 0 1 0; do ML_PKM_BWD_F16=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
k=d.get('kernel_ms_per_step') or {}
print('f16=$c', round(d['ms_per_step'],4), {n: v for n, v in k.items() if 'f16' in n or 'ds_' in n})"; done
for c in 1; do ML_PKM_BWD_F16=$c timeout 300 python scripts/timeline.py > gpurun_out/timeline_f16_$c.txt 2>&1; done
