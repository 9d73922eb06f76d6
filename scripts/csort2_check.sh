# warp-aggregated counting sort + its use in the sparse key backward: parity and A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_large_s.py -q -p no:cacheprovider -x > gpurun_out/cs2_pytest.log 2>&1; echo tests_exit=$?; tail -1 gpurun_out/cs2_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bwd or layer" > gpurun_out/cs2_parity.log 2>&1; echo parity_exit=$?; tail -1 gpurun_out/cs2_parity.log
for cfg in "c3" "c5 --per-rank 8" "c4 --per-rank 8" "c2"; do for c in 1 0 1 0; do ML_SORT_COUNTING=$c timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
k=d['kernel_ms_per_step']
print('$cfg counting=$c', round(d['ms_per_step'],4), {n: v for n, v in k.items() if 'sort' in n or 'run' in n})"; done; done
