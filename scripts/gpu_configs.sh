mkdir -p gpurun_out
for c in c1 c3; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>gpurun_out/bench_$c.err; echo $c exit=$?
python - $c <<'PY'
import json, sys
c = sys.argv[1]
l = [x for x in open(f'gpurun_out/bench_{c}.log') if x.startswith('{')]
if l:
    d = json.loads(l[-1]); print(c, "value", d["value"], "ms", d["ms_per_step"]); print(d["roofline"]); print(d["kernel_ms_per_step"])
else:
    print(open(f'gpurun_out/bench_{c}.err').read()[-2000:])
PY
done
