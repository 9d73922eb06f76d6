# Round-2 profile refresh: plain bench, ncu launch list of the same command,
# ncu --set full of the five hot kernels of the first timed C2 step.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants"
timeout 300 $CMD > gpurun_out/r2p_plain.log 2>&1 && echo plain_ok && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv \
  --log-file gpurun_out/r2p_launches.csv $CMD > gpurun_out/r2p_ncu_launch.log 2>&1; echo launch_exit=$?
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"seg_pipe|bag_fwd_kernel|pkm_scores_tc|half_topk|combine_kernel|pkm_bwd_tc|softmax_bwd|csort_" -s 15 -c 12 \
  -o gpurun_out/r2p_prof $CMD > gpurun_out/r2p_ncu_full.log 2>&1; echo full_exit=$?
tail -n 3 gpurun_out/r2p_ncu_full.log
