mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && echo plain_ok && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_pipe" -s 2 -c 1 -o gpurun_out/prof_pipe $CMD > gpurun_out/ncu_pipe.log 2>&1; echo ncu_exit=$?
tail -3 gpurun_out/ncu_pipe.log
