# half top-k change check: lookup parity tests + bench kernel times + ncu of half_topk alone
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
bash scripts/gpu_ab.sh X=1 2>&1 | grep -v "^$"
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"half_topk|combine_kernel" -s 6 -c 2 --csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E '"(gpu__time|smsp__inst)' | awk -F'","' '{print $5, $(NF-2), $NF}'
