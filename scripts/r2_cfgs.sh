mkdir -p gpurun_out
for cfg in "c4 --per-rank 8" "c5 --per-rank 8" "c3"; do
  tag=$(echo $cfg | cut -d' ' -f1)
  timeout 900 python bench.py --config $cfg --steps 10 --no-cpu-baseline > gpurun_out/r2x_$tag.log 2>&1; echo $tag=$?
done
timeout 600 python bench.py --steps 20 > gpurun_out/r2x_c2.log 2>&1; echo c2=$?
python - <<'PY'
import json
for t in ("c2","c3","c4","c5"):
    f=f"gpurun_out/r2x_{t}.log"
    try:
        d=json.loads([x for x in open(f) if x.startswith('{')][-1])
    except Exception as e:
        print(f, "ERR", e); continue
    print(t, "ms", round(d["ms_per_step"],4), "e2e", round(d["e2e"]["ms_per_step"],3), "bf16dV", (d.get("variants") or {}).get("dV_bf16",{}).get("ms_per_step"), "clk", d["clocks"])
    print("   kern", d["kernel_ms_per_step"])
PY
