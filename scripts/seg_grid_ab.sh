# A/B: the segmented pass's persistent grid sized for fewer SMs (room for the gate GEMMs beside it)
# (the ML_SEG_GRID_SMS switch was removed after this measurement; DESIGN.md §6 has the numbers)
for r in 1 2; do for m in 0 140 128 112; do ML_SEG_GRID_SMS=$m timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('seg_grid_sms=$m', round(d['ms_per_step'],4), d['kernel_ms_per_step'].get('embbag_bwd_segreduce'))"; done; done
