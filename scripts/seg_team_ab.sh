# A/B of the segmented pass's column slicing at C2 (ML_SEG_TEAM=128: two 2 KiB
# slices, slice-major work order) against the default (one 4 KiB slice)
mkdir -p gpurun_out
for t in 256 128 256 128; do ML_SEG_TEAM=$t timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
k=d.get('kernel_ms_per_step') or {}
print('team=$t', round(d['ms_per_step'],4), {n: v for n, v in k.items() if 'seg' in n or 'bag' in n}, d['roofline'].get('avg_ms'))"; done
