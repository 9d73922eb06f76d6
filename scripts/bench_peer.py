"""PEER-style workload timed on one GPU: one step =
peer_fwd + peer_bwd over 16K tokens at the paper's PEER configuration for the
1.3B base (768 half keys -> N = 589,824 experts; expert vectors of the
model dim 2048; 4 heads, k = 32, bf16).  Synthetic inputs; CUDA events around
K steps after W warm-ups.  Prints one JSON line.
    python scripts/bench_peer.py [--steps 10 --warmup 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_09764_b200 import ops  # noqa: E402
from synthetic import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--S", type=int, default=768)
ap.add_argument("--D", type=int, default=2048)
a = ap.parse_args()
S, D, Dk, H, k, T = a.S, a.D, 1024, 4, 32, 16384
dev = torch.device("cuda", 0)
dt = torch.bfloat16


def fill(shape, tag, scale=1.0):
    x = torch.empty(shape, dtype=dt, device=dev)
    ops.synth_fill(x, 0, gen.TAGS[tag], scale=scale)
    return x


x = fill((T, D), "x")
q = fill((T, H, Dk), "q")
K1 = fill((H, S, Dk // 2), "K1", gen.scale_for("K1", Dk=Dk))
K2 = fill((H, S, Dk // 2), "K2", gen.scale_for("K2", Dk=Dk))
U = fill((S * S, D), "W1", gen.scale_for("W1", D=D))
V = fill((S * S, D), "V")
dy = fill((T, D), "dout")
dK1 = torch.zeros(K1.shape, dtype=torch.float32, device=dev)
dK2 = torch.zeros(K2.shape, dtype=torch.float32, device=dev)


def step():
    dK1.zero_()
    dK2.zero_()
    y, saved = ops.peer_fwd(x, q, K1, K2, U, V, k)
    return ops.peer_bwd(dy, x, q, K1, K2, U, V, saved, dK1=dK1, dK2=dK2)


for _ in range(a.warmup):
    g = step()
torch.cuda.synchronize()
ops.timing_reset()
ops.timing_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    g = step()
e1.record()
torch.cuda.synchronize()
ops.timing_enable(False)
kern = ops.timing_report()
ms = e0.elapsed_time(e1) / a.steps
P = T * H * k
print(json.dumps({
    "workload": f"PEER f4: N={S}^2 experts x (U, V in R^{D}), 4 heads, k=32, 16K tokens, bf16",
    "metric": "PEER fwd+bwd tok/s", "value": T / (ms / 1e3), "unit": "tok/s", "ms_per_step": ms,
    "steps": a.steps, "warmup": a.warmup, "unique_rows_per_position": int(g["U"].item()) / P,
    "kernel_ms_per_step": {n: round(v[1] / a.steps, 4) for n, v in sorted(
        kern.items(), key=lambda kv: -kv[1][1])},
    "data": "synthetic"}))
