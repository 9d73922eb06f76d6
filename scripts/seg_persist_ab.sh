# experiment: dy in a persisting L2 window during the segmented pass
# (the ML_SEG_L2_PERSIST switch was removed after this measurement; DESIGN.md §6 has the numbers)
for m in 0 1 48 0 1 48; do echo "ML_SEG_L2_PERSIST=$m"; ML_SEG_L2_PERSIST=$m timeout 300 python scripts/seg_dy_probe.py 2>&1 | grep -v "^$" | head -4; done
for m in 1 0 1 0; do ML_SEG_L2_PERSIST=$m timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('persist=$m', round(d['ms_per_step'],4), d['kernel_ms_per_step'].get('embbag_bwd_segreduce'))"; done
