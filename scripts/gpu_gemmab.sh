# cuBLASLt heuristic-rank A/B: serialised GEMM kernel times of one step per ML_GEMM_ALGO
for v in "$@"; do
  env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"nvjet|gemm|sm100" -s ${S:-20} -c 10 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/gemmab.csv
  python - "$v" <<'PY'
import csv, sys
lines = open('gpurun_out/gemmab.csv').read().splitlines()
i0 = next((i for i, l in enumerate(lines) if l.startswith('"ID"')), None)
if i0 is None: print(sys.argv[1], "no data"); sys.exit()
rows = list(csv.reader(lines[i0:])); h = rows[0]
iN = h.index('Kernel Name'); iV = h.index('Metric Value')
out = [(r[iN][:40], round(float(r[iV].replace(',', '')) / 1e3, 1)) for r in rows[1:]]
print(sys.argv[1], round(sum(v for _, v in out), 1), out)
PY
done
