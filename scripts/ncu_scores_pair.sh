# ncu --set full of the scoring kernel, single CTA vs CTA pair (ML_PKM_PAIR=1), C2
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants"
timeout 900 ncu --set full --clock-control none -k regex:"pkm_scores_tc" -s 3 -c 1 -o gpurun_out/sc_single $CMD > gpurun_out/sc1.log 2>&1; echo single=$?
ML_PKM_PAIR=1 timeout 900 ncu --set full --clock-control none -k regex:"pkm_scores_tc" -s 3 -c 1 -o gpurun_out/sc_pair $CMD > gpurun_out/sc2.log 2>&1; echo pair=$?
