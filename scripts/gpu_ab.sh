# A/B of env switches on the C2 step: bash scripts/gpu_ab.sh "ENV=a" "ENV=b" ...
mkdir -p gpurun_out
for rep in 1 2; do
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python - "$v" <<'PY'
import json,sys
l = [x for x in open('gpurun_out/ab.log') if x.startswith('{')]
if not l: print(sys.argv[1], "FAILED", open('gpurun_out/ab.log').read()[-1500:]); sys.exit()
d = json.loads(l[-1]); k = d["kernel_ms_per_step"]
print(f"{sys.argv[1]:28s} ms {d["ms_per_step"]:.3f} seg {k.get("embbag_bwd_segreduce")} smbwd {k.get("softmax_bwd")} topk {k.get("half_topk")} comb {k.get("combine_softmax")}")
PY
done; done
