# round-2 final config sweep (current tree): every config once, with the bf16-dV variant
mkdir -p gpurun_out
for cfg in "c2" "c2_dv1024" "c2_dv4096" "c3" "c4 --per-rank 8" "c5 --per-rank 8"; do
  tag=$(echo $cfg | cut -d' ' -f1)
  timeout 900 python bench.py --config $cfg --steps 10 --no-cpu-baseline > gpurun_out/r2z_$tag.log 2>gpurun_out/r2z_$tag.err; echo $tag=$?
done
python - <<'PY'
import json
for t in ("c2", "c2_dv1024", "c2_dv4096", "c3", "c4", "c5"):
    f = f"gpurun_out/r2z_{t}.log"
    try:
        d = json.loads([x for x in open(f) if x.startswith('{')][-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k = d["kernel_ms_per_step"]
    print(t, "ms", round(d["ms_per_step"], 4), "tok/s", round(d["value"]), "e2e", round(d["e2e"]["ms_per_step"], 3),
          "bf16dV", (d.get("variants") or {}).get("dV_bf16", {}).get("ms_per_step"), "clk", d["clocks"],
          "frac", d["roofline"]["frac"], "U/P", d["config"].get("unique_rows_per_position"))
    print("   kern", {n: k[n] for n in list(k)[:10]})
PY
