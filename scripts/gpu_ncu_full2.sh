mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && echo plain_ok && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"seg_kernel" -s 3 -c 1 -o gpurun_out/prof_r01b $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_exit=$?
tail -2 gpurun_out/ncu_full.log
