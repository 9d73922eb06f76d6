"""SASS evidence of the Blackwell-native paths (B200_PROFILING.md "What proves
a Blackwell-native kernel"): counts of tcgen05 / TMA / TMEM / bulk-copy /
mbarrier / FFMA2 / 256-bit store mnemonics per kernel of libmemlayer.so.
    python scripts/sass_evidence.py > profiles/r02_sass_evidence.txt
"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "paper_2412_09764_b200", "libmemlayer.so")
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
keys = ["UTCHMMA", "UTCHMMA.2CTA", "UTCBAR", "UTCBAR.2CTA", "LDTM", "UTMALDG", "UTMALDG.2D.2CTA",
        "UTMASTG", "UBLKCP", "SYNCS.ARRIVE",
        "SYNCS.PHASECHK", "FFMA2", "STG.E.ENL2.256", "HMMA", "HGMMA", "LDGSTS"]
cur, ev, arch = None, collections.defaultdict(collections.Counter), set()
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"arch = (sm_\w+)", line)
    if m:
        arch.add(m.group(1))
    ops = re.findall(r"\b([A-Z][A-Z0-9_.]+)\b", line.split(";")[0]) if "/*" in line else []
    for k in keys:
        if any(o == k or o.startswith(k + ".") or (k.endswith(".256") and o == k) for o in ops):
            ev[cur][k] += 1
short = lambda n: re.sub(r"_ZN2ml\d*_GLOBAL__N__\w+?_\d+", "", n)[:70]
print("# cuobjdump -sass paper_2412_09764_b200/libmemlayer.so; arch:", ", ".join(sorted(arch)))
print("# static instruction counts per kernel (mnemonics of B200_PROFILING.md)")
for f in sorted(ev, key=lambda n: short(n)):
    c = {k: v for k, v in ev[f].items() if v}
    if c:
        print(f"{short(f):72s} {c}")
