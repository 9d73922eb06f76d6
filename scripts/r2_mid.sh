mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2u_pytest.log 2>&1; echo pytest_exit=$?
grep -E "passed|failed|FAILED" gpurun_out/r2u_pytest.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2u_smoke.log 2>&1; echo smoke_exit=$?; tail -2 gpurun_out/r2u_smoke.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-group --steps 10 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/r2u_group.log 2>gpurun_out/r2u_group.err; echo group_exit=$?; tail -c 800 gpurun_out/r2u_group.err
timeout 600 python bench.py --steps 20 > gpurun_out/r2u_bench.log 2>gpurun_out/r2u_bench.err; echo bench_exit=$?
timeout 900 python bench.py --config c4 --per-rank 8 --steps 10 --no-cpu-baseline > gpurun_out/r2u_c4.log 2>&1; echo c4=$?
timeout 900 python bench.py --config c5 --per-rank 8 --steps 5 --no-cpu-baseline > gpurun_out/r2u_c5.log 2>&1; echo c5=$?
timeout 900 python bench.py --config c3 --steps 10 --no-cpu-baseline > gpurun_out/r2u_c3.log 2>&1; echo c3=$?
python - <<'PY'
import json
for f in ("gpurun_out/r2u_group.log","gpurun_out/r2u_bench.log","gpurun_out/r2u_c4.log","gpurun_out/r2u_c5.log","gpurun_out/r2u_c3.log"):
    try:
        d=json.loads([x for x in open(f) if x.startswith('{')][-1])
    except Exception as e:
        print(f, "ERR", e); continue
    print(f, "ms", round(d["ms_per_step"],4), "value", round(d["value"]), "e2e", round(d["e2e"]["ms_per_step"],3), "variants", d.get("variants"))
    print("   roof", {k: d["roofline"].get(k) for k in ("kernel","achieved","frac","avg_ms")}, "clocks", d["clocks"])
    print("   kern", d["kernel_ms_per_step"])
    if d.get("collectives"): print("   coll", d["collectives"])
    if d.get("cpu_baseline"): print("   cpu", d["cpu_baseline"]["value"], d["cpu_baseline"].get("single_thread"))
PY
