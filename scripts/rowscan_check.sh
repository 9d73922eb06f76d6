# runs from the counting sort's row scan: bit-identity + C2 A/B against find_runs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py -q -p no:cacheprovider -x > gpurun_out/rs_pytest.log 2>&1; echo sort_exit=$?; tail -2 gpurun_out/rs_pytest.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group_capi.py tests/test_gpu_graph.py -q -p no:cacheprovider -x > gpurun_out/rs_parity.log 2>&1; echo parity_exit=$?; tail -2 gpurun_out/rs_parity.log
for c in 1 0 1 0 1 0 1 0; do ML_RUNS_ROWSCAN=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('rowscan=$c', round(d['ms_per_step'],4))"; done
timeout 300 python scripts/timeline.py > gpurun_out/timeline_rs_1.txt 2>&1
