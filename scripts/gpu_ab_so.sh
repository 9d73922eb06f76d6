# same-box A/B of two library builds: the in-tree libmemlayer.so (new) vs libmemlayer_old.so
# usage: bash scripts/gpu_ab_so.sh <kernel regex>
K=$1
cp paper_2412_09764_b200/libmemlayer.so /tmp/lib_new.so
for v in new old new old; do
  cp /tmp/lib_$v.so paper_2412_09764_b200/libmemlayer.so 2>/dev/null || cp paper_2412_09764_b200/libmemlayer_old.so paper_2412_09764_b200/libmemlayer.so
  [ $v = old ] && cp paper_2412_09764_b200/libmemlayer_old.so paper_2412_09764_b200/libmemlayer.so
  timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"$K" -s ${S:-2} -c ${C:-1} --csv \
    python bench.py --steps 1 --warmup 2 --no-cpu-baseline 2>/dev/null | grep -E '"(gpu__time|smsp__inst)' | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
done
cp /tmp/lib_new.so paper_2412_09764_b200/libmemlayer.so
