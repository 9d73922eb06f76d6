# full round check: tests, smoke, bench (+group path), reference arm, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo bench_exit=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --force-group --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_group.log 2>gpurun_out/bench_group.err; echo group_bench_exit=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>gpurun_out/bench_ref.err; echo ref_exit=$?
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && echo plain_ok && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu_exit=$?
python - <<'PY'
import json
for f in ("gpurun_out/bench.log", "gpurun_out/bench_group.log", "gpurun_out/bench_ref.log"):
    l = [x for x in open(f) if x.startswith('{')]
    if not l:
        print(f, "NO JSON"); continue
    d = json.loads(l[-1])
    print(f, "value", d.get("value"), "ms", d.get("ms_per_step"), "e2e", (d.get("e2e") or {}).get("value"))
    print("  roofline", d.get("roofline")); print("  cpu", d.get("cpu_baseline")); print("  clocks", d.get("clocks"), "launches", d.get("gpu_launches"))
PY
tail -n 3 gpurun_out/bench.err gpurun_out/bench_group.err gpurun_out/bench_ref.err
