"""Summarise an ncu source page (SASS): totals, stall mix, hottest lines."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed")
totE = sum(int(r[iE]) for r in data); totS = sum(int(r[iS]) for r in data)
print("warp instr total", totE, "samples", totS)
names = [n for n in h if n.startswith('stall_') and '(' not in n]
tot = {n: sum(int(r[h.index(n)] or 0) for r in data) for n in names}
T = sum(tot.values()) or 1
print({n[6:]: round(v / T, 3) for n, v in sorted(tot.items(), key=lambda x: -x[1])[:8]})
N = int(sys.argv[2]) if len(sys.argv) > 2 else 15
for r in sorted(data, key=lambda r: -int(r[iS]))[:N]:
    print(r[0][-5:], r[1][:70], r[iS], r[iE])
