mkdir -p gpurun_out
cp paper_2412_09764_b200/libmemlayer.so /tmp/lib_keep.so
for v in 16 8 12 24 16 8 12 24; do
  cp paper_2412_09764_b200/_ab/lib_$v.so paper_2412_09764_b200/libmemlayer.so
  t=$(timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sort_scatter" -s 2 -c 2 --csv \
    python bench.py --steps 1 --warmup 2 --no-cpu-baseline 2>/dev/null | grep -E '"gpu__time' | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}')
  ms=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; print(json.loads(sys.stdin.read().strip().splitlines()[-1])['ms_per_step'])")
  echo "rounds=$v scatter_ns=[$t] step_ms=$ms"
done
cp /tmp/lib_keep.so paper_2412_09764_b200/libmemlayer.so
