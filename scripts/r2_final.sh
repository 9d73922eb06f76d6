# round-2 end-state check: GPU suite, smoke, default bench, reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2f_pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/r2f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo smoke_exit=$?; tail -3 gpurun_out/r2f_smoke.log
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2>gpurun_out/r2f_bench.err; echo bench_exit=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_ref.log 2>gpurun_out/r2f_ref.err; echo ref_exit=$?
python - <<'PY'
import json
for f in ("gpurun_out/r2f_bench.log", "gpurun_out/r2f_ref.log"):
    l = [x for x in open(f) if x.startswith('{')]
    d = json.loads(l[-1])
    print(f, "value", d.get("value"), "ms", d.get("ms_per_step"), "e2e", (d.get("e2e") or {}).get("ms_per_step"),
          "clocks", d.get("clocks"), "launches", d.get("gpu_launches"))
    print("  roofline", {k: d.get("roofline", {}).get(k) for k in ("kernel", "frac", "achieved", "traffic")} if d.get("roofline") else None)
    print("  variants", d.get("variants"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
PY
