mkdir -p gpurun_out
for mb in 0 48 80; do
ML_L2_PERSIST_MB=$mb timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_l2_$mb.log 2>&1
python -c "
import json
d=json.loads([x for x in open('gpurun_out/bench_l2_$mb.log') if x.startswith('{')][-1]); print('$mb', d['ms_per_step'], d['kernel_ms_per_step']['embbag_bwd_segreduce'])"
done
