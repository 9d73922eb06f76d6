# 8-element register network in the counting sort's fixup: tests + csort_fix times
timeout 900 python -m pytest tests/test_gpu_sort.py -q -p no:cacheprovider -x 2>&1 | tail -1
for cfg in "c4 --per-rank 8" "c2"; do for r in 1 2; do timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
k=d['kernel_ms_per_step']
print('$cfg', round(d['ms_per_step'],4), {n: v for n, v in k.items() if 'csort' in n})"; done; done
