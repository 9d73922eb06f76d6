# round-2 check: full GPU suite, smoke, bench (C2), per-rank C4/C5 lines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2b_pytest_gpu.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/r2b_pytest_gpu.log | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo smoke_exit=$?; tail -3 gpurun_out/r2b_smoke.log
timeout 600 python bench.py > gpurun_out/r2b_bench.log 2>gpurun_out/r2b_bench.err; echo bench_exit=$?; tail -c 1500 gpurun_out/r2b_bench.err
timeout 900 python bench.py --config c4 --per-rank 8 --steps 10 --no-cpu-baseline > gpurun_out/r2b_c4_pr8.log 2>gpurun_out/r2b_c4_pr8.err; echo c4_exit=$?; tail -c 1500 gpurun_out/r2b_c4_pr8.err
timeout 900 python bench.py --config c5 --per-rank 8 --steps 5 --no-cpu-baseline > gpurun_out/r2b_c5_pr8.log 2>gpurun_out/r2b_c5_pr8.err; echo c5_exit=$?; tail -c 1500 gpurun_out/r2b_c5_pr8.err
python - <<'PY'
import json
for f in ("gpurun_out/r2b_bench.log", "gpurun_out/r2b_c4_pr8.log", "gpurun_out/r2b_c5_pr8.log"):
    try:
        l = [x for x in open(f) if x.startswith('{')]
    except Exception as e:
        print(f, e); continue
    if not l:
        print(f, "NO JSON"); continue
    d = json.loads(l[-1])
    print(f, "value", d.get("value"), "ms", d.get("ms_per_step"), "e2e", (d.get("e2e") or {}).get("ms_per_step"))
    print("  roofline", d.get("roofline")); print("  scoring", d.get("scoring_roofline"))
    print("  kern", d.get("kernel_ms_per_step")); print("  cpu", d.get("cpu_baseline")); print("  clocks", d.get("clocks"), "launches", d.get("gpu_launches"))
PY
