# same-box A/B of two library builds on the scoring kernel (libmemlayer.so = new, libmemlayer_old.so = old)
cp paper_2412_09764_b200/libmemlayer.so /tmp/lib_new.so
for v in new old new old new old; do
  if [ $v = old ]; then cp paper_2412_09764_b200/libmemlayer_old.so paper_2412_09764_b200/libmemlayer.so; else cp /tmp/lib_new.so paper_2412_09764_b200/libmemlayer.so; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-variants > gpurun_out/ab.log 2>&1
  python - $v <<'PY'
import json, sys
l = [x for x in open('gpurun_out/ab.log') if x.startswith('{')]
d = json.loads(l[-1]); k = d["kernel_ms_per_step"]
print(sys.argv[1], "ms", round(d["ms_per_step"], 4), "scores", k.get("pkm_scores_tc"), "topk", k.get("half_topk"))
PY
done
cp /tmp/lib_new.so paper_2412_09764_b200/libmemlayer.so
