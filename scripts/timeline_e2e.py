"""Timeline of bench.py's e2e loop (host inputs, copy streams) via
torch.profiler: per-op start/duration/stream for the last step.  Diagnostic."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2412_09764_b200 import ops  # noqa: E402


class A:
    steps = 6
    no_state = "--no-state" in sys.argv


cfg = bench.CONFIGS["c2"]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
t = bench.make_inputs(cfg, dev, 1, 0, ops, torch)
k = cfg["k"]
dK1 = torch.zeros(t["K1"].shape, dtype=torch.float32, device=dev)
dK2 = torch.zeros(t["K2"].shape, dtype=torch.float32, device=dev)
bufs = {}


def step(inp=t):
    dK1.zero_()
    dK2.zero_()
    out, saved = ops.memory_layer_fwd(inp["x"], inp["q"], t["K1"], t["K2"], t["V"], t["W1"],
                                      t["W2"], k, keep_state=not A.no_state)
    g = ops.memory_layer_bwd(inp["dout"], inp["x"], inp["q"], t["K1"], t["K2"], t["V"], t["W1"],
                             t["W2"], saved, dK1=dK1, dK2=dK2, bufs=bufs)
    return out, g


for _ in range(3):
    step()
torch.cuda.synchronize()
stream = torch.cuda.current_stream()
print("compute stream", stream.cuda_stream)
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    r = bench.run_e2e(A, t, step, stream, torch, cfg, 1, 1)
print("e2e", r["ms_per_step"])
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ks = sorted((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0), e.name)
            for e in ev)
t0 = ks[0][0]
for s, e, sid, name in ks:
    if e - s > 20 or "emcpy" in name:
        print(f"{(s - t0) / 1000:9.3f} ms {(e - s) / 1000:7.3f} ms  s{sid:<4d} {name[:70]}")
