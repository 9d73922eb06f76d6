"""Per-rank bag kernels at the 8-GPU memory-group shape (C4: N = 8192^2,
dv = 2048 sharded 8 ways -> 256-column slices; every rank runs the bag over
all 8 x 16K tokens).  Times embbag_fwd and embbag_bwd alone (torch.profiler
kernel sums).  Diagnostic only: python scripts/probe_g8.py [--G 8]"""
import argparse
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_09764_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--G", type=int, default=8)
ap.add_argument("--S", type=int, default=8192)
a = ap.parse_args()
dev = torch.device("cuda", 0)
N, dv, T, B = a.S * a.S, 2048 // a.G, 16384 * a.G, 128
g = torch.Generator(device=dev).manual_seed(0)
idx = torch.randint(0, N, (T, B), dtype=torch.int32, device=dev, generator=g)
w = torch.rand((T, B), device=dev, generator=g)
dy = torch.randn((T, dv), device=dev, generator=g).to(torch.bfloat16)
V = torch.empty((N, dv), device=dev, dtype=torch.bfloat16)
V.normal_(generator=g)
for _ in range(2):
    ops.embbag_fwd(V, idx, w)
    ops.embbag_bwd(V, idx, w, dy, sync=False)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        ops.embbag_fwd(V, idx, w)
        r = ops.embbag_bwd(V, idx, w, dy, sync=False)
    torch.cuda.synchronize()
tot = defaultdict(float)
for e in prof.events():
    if e.device_type.name == "CUDA":
        tot[e.name.replace("ml::(anonymous namespace)::", "")[:60]] += (e.time_range.end - e.time_range.start) / 3
print(f"G={a.G} N={N} dv_local={dv} T_all={T} P={T*B} U/P={int(r[2].item())/(T*B):.3f}")
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:9.1f} us  {n}")
print(f"total {sum(tot.values()):.1f} us")
