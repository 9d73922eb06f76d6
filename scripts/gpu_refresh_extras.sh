# refresh the f-row and group records with the current kernels
mkdir -p gpurun_out
timeout 600 python bench.py --qk-norm --no-cpu-baseline > gpurun_out/bench_qknorm.log 2>&1; echo qk_exit=$?
grep '^{' gpurun_out/bench_qknorm.log | tail -n 1 > gpurun_out/bench_qknorm.jsonl
timeout 600 python scripts/bench_f1.py > gpurun_out/f1.log 2>&1; echo f1_exit=$?
tail -n 1 gpurun_out/f1.log
bash scripts/gpu_group2.sh
grep '^{' gpurun_out/bench_group.log | tail -n 1 > gpurun_out/bench_group.jsonl
