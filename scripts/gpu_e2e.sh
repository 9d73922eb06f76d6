mkdir -p gpurun_out
python scripts/h2d_probe.py 2>&1 | tail -6
for f in "" "--no-state"; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $f > gpurun_out/bench_e2e.log 2>&1
python - <<'PY'
import json
l = [x for x in open('gpurun_out/bench_e2e.log') if x.startswith('{')]
d = json.loads(l[-1]); print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"])
PY
done
