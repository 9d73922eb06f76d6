# round-2: large-S configs after the chunk-filtered half top-k
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_large_s.py -q -x -p no:cacheprovider -k chunk 2>&1 | tail -1
run() {  # name args...
  n=$1; shift
  timeout 900 python bench.py "$@" --no-cpu-baseline --no-variants > gpurun_out/r2c_$n.log 2>gpurun_out/r2c_$n.err; echo $n exit=$?
  python - "$n" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/r2c_{sys.argv[1]}.log") if x.startswith('{')]
d = json.loads(l[-1])
print(sys.argv[1], "ms", d.get("ms_per_step"), "value", round(d.get("value")), "e2e", (d.get("e2e") or {}).get("ms_per_step"), "clocks", d.get("clocks"))
print("  kern", d.get("kernel_ms_per_step"))
PY
}
run c3 --config c3 --steps 10
run c4 --config c4 --per-rank 8 --steps 10
run c5 --config c5 --per-rank 8 --steps 5
