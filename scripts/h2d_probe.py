# raw pinned host->device copy bandwidth on this box (1, 2, 4 streams)
import time, torch
n = 256 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    ch = n // ns
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i*ch:(i+1)*ch].copy_(h[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize(); el = time.perf_counter() - t
    print(f"H2D streams={ns}: {n/el/1e9:.1f} GB/s")
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    h2.copy_(d, non_blocking=True); torch.cuda.synchronize(); el = time.perf_counter() - t
print(f"D2H: {n/el/1e9:.1f} GB/s")
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max", "--format=csv"], capture_output=True, text=True).stdout)
