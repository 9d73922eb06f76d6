mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && echo plain_ok && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"seg_kernel|bag_fwd_kernel|pkm_scores_tc|half_topk|combine" -s 9 -c 9 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_exit=$?
tail -5 gpurun_out/ncu_full.log
