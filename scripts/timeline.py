"""Kernel timeline of one C2 bench step (torch.profiler / CUPTI): per-kernel
start, duration and stream, plus idle gaps of the device.  Diagnostic only.

    python scripts/timeline.py [--keep-state 0|1] > gpurun_out/timeline.txt
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import bench  # noqa: E402
from paper_2412_09764_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--keep-state", type=int, default=1)
ap.add_argument("--config", default="c2")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
t = bench.make_inputs(cfg, dev, 1, 0, ops, torch, False)
k = cfg["k"]
dK1 = torch.zeros(t["K1"].shape, dtype=torch.float32, device=dev)
dK2 = torch.zeros(t["K2"].shape, dtype=torch.float32, device=dev)
bufs = {}


def step():
    dK1.zero_()
    dK2.zero_()
    out, saved = ops.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"],
                                      k, keep_state=bool(a.keep_state))
    g = ops.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"],
                             t["W2"], saved, dK1=dK1, dK2=dK2, bufs=bufs)
    return out, g


for _ in range(4):
    step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ks = []
for e in ev:
    tr = e.time_range
    ks.append((tr.start, tr.end, getattr(e, "device_resource_id", 0), e.name))
ks.sort()
# the last step: from the last "memset"/first kernel after 2/3 of the events
n = len(ks) // 3
last = ks[2 * n:]
t0 = last[0][0]
print(f"# kernels in last step: {len(last)}")
print("# start_us  dur_us  stream  name")
for s, e, sid, name in last:
    print(f"{s - t0:9.1f} {e - s:8.1f} {sid:6d}  {name[:90]}")
# union busy time and gaps
iv = sorted((s, e) for s, e, _, _ in last)
busy, cur_s, cur_e, gaps = 0.0, iv[0][0], iv[0][1], []
for s, e in iv[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((cur_e - t0, s - cur_e))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
span = cur_e - t0
print(f"# span {span:.1f} us, busy {busy:.1f} us, idle {span - busy:.1f} us")
for at, g in sorted(gaps, key=lambda x: -x[1])[:10]:
    print(f"# gap at {at:9.1f} us: {g:.1f} us")
