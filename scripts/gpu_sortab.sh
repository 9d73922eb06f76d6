# sort-pass A/B: serialised kernel time of the state build (sort + runs) per variant
for v in "$@"; do
  env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sort_|run_|scan_" -s 60 -c 40 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/sortab.csv
  python - "$v" <<'PY'
import csv, sys, io
lines = open('gpurun_out/sortab.csv').read().splitlines()
i0 = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[i0:]))
h = rows[0]; iN = h.index('Kernel Name'); iV = h.index('Metric Value'); iI = h.index('ID')
seen = []
tot = 0.0
ks = {}
for r in rows[1:]:
    try: v = float(r[iV].replace(',', ''))
    except: continue
    name = r[iN].split('(')[0].split('::')[-1]
    ks.setdefault(name, []).append(v / 1e3)
print(sys.argv[1], {k: [round(x, 1) for x in v[:6]] for k, v in ks.items()})
PY
done
