# A/B: the forward's value-row state build on the high-priority aux 1
# (ML_STATE_STREAM=1) vs the normal-priority aux 2 (default)
mkdir -p gpurun_out
for c in 1 2 1 2 1 2 1 2; do ML_STATE_STREAM=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('state_stream=$c', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4))"; done
ML_STATE_STREAM=1 timeout 300 python scripts/timeline.py > gpurun_out/timeline_ss_1.txt 2>&1
