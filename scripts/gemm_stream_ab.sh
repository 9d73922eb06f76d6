# A/B: the layer backward's gate GEMMs on a normal-priority stream (default)
# vs the high-priority aux 1 (ML_BWD_GEMM_STREAM=1)
mkdir -p gpurun_out
for c in 4 1 4 1 4 1 4 1; do ML_BWD_GEMM_STREAM=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('gemm_stream=$c', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4))"; done
for c in 4 1; do ML_BWD_GEMM_STREAM=$c timeout 300 python scripts/timeline.py > gpurun_out/timeline_gs_$c.txt 2>&1; done
