mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2d_pytest.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|FAILED" gpurun_out/r2d_pytest.log | tail -12
timeout 600 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/r2d_bench.log 2>gpurun_out/r2d_bench.err; echo bench_exit=$?; tail -c 600 gpurun_out/r2d_bench.err
timeout 900 python bench.py --config c4 --per-rank 8 --steps 10 --no-cpu-baseline > gpurun_out/r2d_c4.log 2>gpurun_out/r2d_c4.err; echo c4_exit=$?
timeout 900 python bench.py --config c5 --per-rank 8 --steps 5 --no-cpu-baseline > gpurun_out/r2d_c5.log 2>gpurun_out/r2d_c5.err; echo c5_exit=$?; tail -c 600 gpurun_out/r2d_c5.err
python - <<'PY'
import json
for f in ("gpurun_out/r2d_bench.log", "gpurun_out/r2d_c4.log", "gpurun_out/r2d_c5.log"):
    try:
        d = json.loads([x for x in open(f) if x.startswith('{')][-1])
    except Exception as e:
        print(f, "ERR", e); continue
    print(f, "ms", round(d["ms_per_step"],4), "variants", d.get("variants"))
    print("  kern", d.get("kernel_ms_per_step"))
PY
