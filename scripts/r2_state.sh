# round-2: group state built once per group -- tests + per-rank C4/C5 kernel lists
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_group_capi.py tests/test_gpu_group.py -q -x -p no:cacheprovider 2>&1 | tail -3
for c in "c4 10" "c5 5"; do set -- $c
  timeout 900 python bench.py --config $1 --per-rank 8 --steps $2 --no-cpu-baseline --no-variants > gpurun_out/r2s_$1.log 2>gpurun_out/r2s_$1.err; echo $1 exit=$?
  python - "$1" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/r2s_{sys.argv[1]}.log") if x.startswith('{')]
d = json.loads(l[-1])
print(sys.argv[1], "ms", d.get("ms_per_step"), "e2e", (d.get("e2e") or {}).get("ms_per_step"), "clocks", d.get("clocks"))
print("  kern", d.get("kernel_ms_per_step"))
PY
done
