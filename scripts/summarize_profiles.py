"""Turn the round's ncu outputs (scripts/gpu_profiles.sh) into the committed
summaries under profiles/:
  profiles/<tag>_launches.txt  - the launch list of one bench command
                                 (cold-cache, serialised ncu durations) and
                                 each kernel's share of one steady-state step
  profiles/<tag>_ncu_summary.txt - ncu --set full of the hot kernels
  profiles/traffic.json        - DRAM bytes per launch of those kernels (C2)
    python scripts/summarize_profiles.py r01 gpurun_out/launches.csv gpurun_out/prof_round.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]

LABEL = OrderedDict([("seg_pipe_kernel", "embbag_bwd_segreduce"),
                     ("bag_fwd_kernel", "embbag_fwd_gate"),
                     ("pkm_scores_tc_kernel", "pkm_scores_tc"),
                     ("half_topk_kernel", "half_topk"),
                     ("combine_kernel", "combine_softmax"),
                     ("pkm_bwd_tc_kernel", "pkm_dq_tc / pkm_dK_tc")])


def short(name):
    n = name.replace("void ", "")
    for pre in ("ml::<unnamed>::", "ml::(anonymous namespace)::", "unnamed>::"):
        n = n.replace(pre, "")
    return n.split("(")[0][:60]


# ---- launch list
rows = [r for r in csv.reader(l for l in open(launches) if l.startswith('"'))]
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
ks = [(short(r[ik]), float(r[iv]) / 1e3) for r in rows[1:]]
# one steady-state step: the launches between the 4th and 5th pkm_scores_tc
# (warmup 3 + first timed step)
starts = [i for i, (n, _) in enumerate(ks) if n.startswith("pkm_scores_tc_kernel")]
a, b = starts[3], starts[4]
step = ks[a:b]
tot = sum(t for _, t in step)
out = io.StringIO()
out.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold cache, serialised)\n")
out.write(f"# command: python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants ; {len(ks)} launches\n")
out.write(f"# one steady-state step = launches {a}..{b - 1}: {len(step)} launches, {tot:.1f} us serialised\n")
out.write("# us        share  kernel\n")
for n, t in step:
    out.write(f"{t:10.1f}  {t / tot:6.3f}  {n}\n")
agg = OrderedDict()
for n, t in step:
    agg[n] = agg.get(n, 0.0) + t
out.write("\n# per kernel (sum over the step)\n")
for n, t in sorted(agg.items(), key=lambda x: -x[1]):
    out.write(f"{t:10.1f}  {t / tot:6.3f}  {n}\n")
out.write("\n# full launch list\n")
for i, (n, t) in enumerate(ks):
    out.write(f"{i:4d} {t:10.1f}  {n}\n")
open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w").write(out.getvalue())

# ---- ncu --set full summary
mets = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_issued.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__registers_per_thread"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(mets)],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hh = r[0]
ix = {m: hh.index(m) for m in mets}
ikn = hh.index("Kernel Name")
units = {m: r[1][ix[m]] for m in mets}
out = io.StringIO()
out.write("# ncu --set full --clock-control none, one launch per kernel of a steady-state C2 step\n")
out.write("# kernel | ms | DRAM read GB | DRAM write GB | DRAM TB/s | % of 6551 GB/s | L2 hit % | "
          "warps active % | issue active % | grid | regs\n")
traffic = {}
for x in r[2:]:
    name = short(x[ikn])
    ms = float(x[ix["gpu__time_duration.sum"]])
    if units["gpu__time_duration.sum"] == "us":
        ms /= 1e3
    rd = float(x[ix["dram__bytes_read.sum"]])
    wr = float(x[ix["dram__bytes_write.sum"]])
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rd *= scale[units["dram__bytes_read.sum"]]
    wr *= scale[units["dram__bytes_write.sum"]]
    tbs = (rd + wr) / (ms / 1e3) / 1e12
    out.write(f"{name:40s} | {ms:7.3f} | {rd / 1e9:7.3f} | {wr / 1e9:7.3f} | {tbs:5.2f} | "
              f"{tbs * 1e3 / 6551.4 * 100:5.1f} | {float(x[ix['lts__t_sector_hit_rate.pct']]):5.1f} | "
              f"{float(x[ix['sm__warps_active.avg.pct_of_peak_sustained_active']]):5.1f} | "
              f"{float(x[ix['sm__inst_issued.avg.pct_of_peak_sustained_active']]):5.1f} | "
              f"{x[ix['launch__grid_size']]} | {x[ix['launch__registers_per_thread']]}\n")
    for key, lab in LABEL.items():
        if name.startswith(key):
            traffic[lab] = int(rd + wr)
# tensor-pipe utilisation of the tcgen05 scoring kernel (a1)
tmets = ["sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
         "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
         "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]
rawt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rt = list(csv.reader(io.StringIO(rawt)))
tutil = {}
for x in rt[2:]:
    nm = short(x[rt[0].index("Kernel Name")])
    if nm.startswith("pkm_scores_tc"):
        vals = {}
        for m in tmets:
            if m in rt[0]:
                try:
                    vals[m.split(".", 2)[-1] if m.startswith("TPC") else m] = float(
                        x[rt[0].index(m)].replace(",", ""))
                except ValueError:
                    pass
        tutil["pkm_scores_tc"] = vals
        out.write(f"\n# {nm}: tensor pipe " + ", ".join(f"{k} = {v:.1f} %" for k, v in vals.items()) + "\n")
if tutil:
    tu = os.path.join(ROOT, "profiles", "tensor_util.json")
    json.dump({"_note": f"ncu --set full (profiles/{tag}_ncu_summary.txt), C2", "c2": tutil},
              open(tu, "w"), indent=1, sort_keys=True)
open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.txt"), "w").write(out.getvalue())
tf = os.path.join(ROOT, "profiles", "traffic.json")
allt = json.load(open(tf)) if os.path.exists(tf) else {}
allt["c2"] = traffic
allt["_note"] = ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch from "
                 f"profiles/{tag}_ncu_summary.txt (ncu --set full, C2)")
json.dump(allt, open(tf, "w"), indent=1, sort_keys=True)
print(open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.txt")).read())
print("\n".join(open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt")).read().split("\n")[:60]))
