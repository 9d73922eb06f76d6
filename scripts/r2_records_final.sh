# round-2 end records at the current tree: config sweep, profile refresh (launch list +
# ncu full), one C4 per-rank launch list
bash scripts/r2_sweep_final.sh
bash scripts/gpu_profiles_r2.sh
CMD4="python bench.py --config c4 --per-rank 8 --steps 2 --warmup 3 --no-cpu-baseline --no-variants"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3200 --csv \
  --log-file gpurun_out/r2p_c4_launches.csv $CMD4 > gpurun_out/r2p_c4_ncu.log 2>&1; echo c4_launch_exit=$?
