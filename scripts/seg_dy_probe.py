"""Diagnostic: the segmented backward at C2's positions (P = 2.1M over 2^20
rows, dv = 2048 bf16) with the dy rows spread over T = 16384 tokens (64 MiB,
C2) vs T = 2048 tokens (8 MiB, fits L2 many times over): the difference is
the cost of dy rows the L2 does not keep.  python scripts/seg_dy_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2412_09764_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
N, dv, P = 1 << 20, 2048, 16384 * 128
g = torch.Generator(device=dev).manual_seed(0)
V = torch.randn((N, dv), device=dev, generator=g).to(torch.bfloat16)
for T in (16384, 4096, 2048):
    B = P // T
    idx = torch.randint(0, N, (T, B), dtype=torch.int32, device=dev, generator=g)
    w = torch.rand((T, B), device=dev, generator=g)
    dy = torch.randn((T, dv), device=dev, generator=g).to(torch.bfloat16)
    st = ops.embbag_bwd_prepare(N, dv, idx)
    bufs = {}
    for _ in range(3):
        ops.embbag_bwd(V, idx, w, dy, sync=False, state=st, bufs=bufs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ops.embbag_bwd(V, idx, w, dy, sync=False, state=st, bufs=bufs)
    e1.record()
    torch.cuda.synchronize()
    print(f"T={T} B={B} dy={T * dv * 2 / 2**20:.0f} MiB: {e0.elapsed_time(e1) / 10:.3f} ms per backward")
