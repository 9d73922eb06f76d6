import sys, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2412_09764_b200 import ops
cfg = bench.CONFIGS["c2"]
dev = torch.device("cuda", 0)
t = bench.make_inputs(cfg, dev, 1, 0, ops, torch, False)
idx, w = ops.pkm_topk(t["q"], t["K1"], t["K2"], cfg["k"])
c = torch.bincount(idx.flatten().long(), minlength=cfg["S"] ** 2)
nz = c[c > 0]
print("P", idx.numel(), "U", nz.numel(), "max run", int(nz.max()), "runs>32", int((nz > 32).sum()), "runs>256", int((nz > 256).sum()), "positions in runs>32", int(nz[nz > 32].sum()))
for q in (0.5, 0.9, 0.99, 0.999):
    print(q, float(torch.quantile(nz.float(), q)))
