# usage: KREGEX=half_topk bash scripts/gpu_ncu_kernel.sh
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && echo plain_ok && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s 1 -c 1 -o gpurun_out/prof_k $CMD > gpurun_out/ncu_k.log 2>&1; echo ncu_exit=$?
tail -2 gpurun_out/ncu_k.log
