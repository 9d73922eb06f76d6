# softmax-backward change check: parity subset + ncu time/instructions of softmax_bwd
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pkm or layer or qk or peer or autograd" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"softmax_bwd" -s 2 -c 1 --csv \
  python bench.py --steps 1 --warmup 2 --no-cpu-baseline 2>/dev/null | grep -E '"(gpu__time|smsp__inst)' | awk -F'","' '{print $(NF-2), $NF}'
