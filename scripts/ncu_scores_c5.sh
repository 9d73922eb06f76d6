# ncu --set full of the scoring kernel at the C5 per-rank shape (S = 8192, Dh = 1024)
mkdir -p gpurun_out
CMD="python bench.py --config c5 --per-rank 8 --steps 1 --warmup 3 --no-cpu-baseline --no-variants"
timeout 600 $CMD > gpurun_out/c5s_plain.log 2>&1 && echo plain_ok
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pkm_scores_tc" -s 3 -c 1 \
  -o gpurun_out/c5_scores $CMD > gpurun_out/c5s_ncu.log 2>&1; echo ncu_exit=$?
