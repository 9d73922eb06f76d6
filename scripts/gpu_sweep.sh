mkdir -p gpurun_out
: > gpurun_out/bench_sweep.jsonl
for c in c2 c2_dv1024 c2_dv4096 c3; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>gpurun_out/bench_$c.err; echo $c exit=$?
grep '^{' gpurun_out/bench_$c.log | tail -n 1 >> gpurun_out/bench_sweep.jsonl
python - $c <<'PY'
import json, sys
c = sys.argv[1]
l = [x for x in open(f'gpurun_out/bench_{c}.log') if x.startswith('{')]
if l:
    d = json.loads(l[-1]); print(c, "value", round(d["value"]), "ms", round(d["ms_per_step"], 3), "bag", {k: (v["avg_ms"], v["frac"]) for k, v in d["bag_kernels"].items()})
else:
    print(open(f'gpurun_out/bench_{c}.err').read()[-2000:])
PY
done
