"""Kernel times of the bag backward alone (sort + runs + segmented
reduction) on C2-shaped indices, via torch.profiler.  Diagnostic only."""
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_09764_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
N, dv, T, B = 1 << 20, int(os.environ.get("DV", "2048")), 16384, 128
g = torch.Generator(device=dev).manual_seed(0)
idx = torch.randint(0, N, (T, B), dtype=torch.int32, device=dev, generator=g)
w = torch.rand((T, B), device=dev, generator=g)
dy = torch.randn((T, dv), device=dev, generator=g).to(torch.bfloat16)
V = torch.randn((N, dv), device=dev, generator=g).to(torch.bfloat16)
for _ in range(3):
    ops.embbag_bwd(V, idx, w, dy, sync=False)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        ops.embbag_bwd(V, idx, w, dy, sync=False)
    torch.cuda.synchronize()
tot = defaultdict(float)
for e in prof.events():
    if e.device_type.name == "CUDA":
        tot[e.name.replace("ml::(anonymous namespace)::", "")[:60]] += (e.time_range.end - e.time_range.start) / 5
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:9.1f} us  {n}")
