"""Read-only vs copy HBM bandwidth on this GPU (torch kernels; diagnostic)."""
import torch
n = 4 << 30   # 4 Gi bf16 elements = 8 GiB
a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
a.fill_(1)
b = torch.empty(n // 4, dtype=torch.bfloat16, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
ms = t(lambda: a.view(-1, 4096).amax(dim=1))
print(f"read 8 GiB (amax rows): {ms:.3f} ms = {8 * 2**30 / ms / 1e6:.0f} GB/s")
ms = t(lambda: a.sum())
print(f"read 8 GiB (sum): {ms:.3f} ms = {8 * 2**30 / ms / 1e6:.0f} GB/s")
src = a[: n // 4]
ms = t(lambda: b.copy_(src))
print(f"copy 2 GiB: {ms:.3f} ms = {2 * 2 * 2**30 / ms / 1e6:.0f} GB/s (r+w)")
