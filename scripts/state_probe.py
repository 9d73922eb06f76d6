"""The memory group's backward state at a per-rank shape: one sort of all
G*T_loc*B gathered positions (embbag_bwd_prepare, round 1) vs the
once-per-group build (own positions sorted, G sorted lists merged:
embbag_bwd_group_sort_local + embbag_bwd_group_merge).  Per-kernel times
from the library's timing marks (one stream).  Diagnostic only:
python scripts/state_probe.py [--G 8] [--S 8192] [--T 2048]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_09764_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--G", type=int, default=8)
ap.add_argument("--S", type=int, default=8192)
ap.add_argument("--T", type=int, default=2048, help="tokens per rank")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
dev = torch.device("cuda", 0)
N, B, G, T = a.S * a.S, 128, a.G, a.T
g = torch.Generator(device=dev).manual_seed(0)
idx_all = torch.randint(0, N, (G * T, B), dtype=torch.int32, device=dev, generator=g)
lists = torch.empty((G, 2, T * B), dtype=torch.int32, device=dev)
for r in range(G):
    ops.group_sort_local(N, idx_all[r * T:(r + 1) * T], r, out=lists[r])
own = idx_all[:T].contiguous()
lst = torch.empty((2, T * B), dtype=torch.int32, device=dev)
st_old = ops.embbag_bwd_prepare(N, 256, idx_all)
st_new = ops.group_merge(N, 256, lists)
ws = None


def old():
    ops.embbag_bwd_prepare(N, 256, idx_all, out=st_old)


def new():
    ops.group_sort_local(N, own, 0, out=lst)
    ops.group_merge(N, 256, lists, out=st_new)


for name, fn in (("one sort of all positions", old), ("own sort + merge", new)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ops.timing_reset()
    ops.timing_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ops.timing_enable(False)
    rep = ops.timing_report()
    print(f"{name}: {e0.elapsed_time(e1) / a.reps:.4f} ms  per kernel:",
          {n: round(v[1] / a.reps, 4) for n, v in sorted(rep.items(), key=lambda kv: -kv[1][1])})

# kernel durations (CUPTI), independent of the host's launch rate
from collections import defaultdict  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402
for name, fn in (("one sort of all positions", old), ("own sort + merge", new)):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            fn()
        torch.cuda.synchronize()
    tot = defaultdict(float)
    for e in prof.events():
        if e.device_type.name == "CUDA":
            tot[e.name.replace("ml::(anonymous namespace)::", "")[:48]] += \
                (e.time_range.end - e.time_range.start) / a.reps
    print(f"{name} (CUPTI kernel us, sum {sum(tot.values()):.1f}):",
          {n: round(v, 1) for n, v in sorted(tot.items(), key=lambda x: -x[1])})
