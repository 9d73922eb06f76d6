"""pkm_topk_bwd at C2/C3 per-head shapes: per-kernel times (probe)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2412_09764_b200 import ops
from synthetic import gen
T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
H, Dk, k = 4, 1024, 32
q = torch.empty((T, H, Dk), dtype=torch.bfloat16, device="cuda")
K1 = torch.empty((H, S, Dk // 2), dtype=torch.bfloat16, device="cuda")
K2 = torch.empty_like(K1)
ops.synth_fill(q, 0, gen.TAGS["q"])
ops.synth_fill(K1, 0, gen.TAGS["K1"], scale=gen.scale_for("K1", Dk=Dk))
ops.synth_fill(K2, 0, gen.TAGS["K2"], scale=gen.scale_for("K2", Dk=Dk))
idx, w = ops.pkm_topk(q, K1, K2, k)
dw = torch.randn((T, H, k), device="cuda")
dK1 = torch.zeros(K1.shape, device="cuda"); dK2 = torch.zeros(K2.shape, device="cuda")
for _ in range(3):
    ops.pkm_topk_bwd(q, K1, K2, idx, w, dw, dK1, dK2)
torch.cuda.synchronize()
ops.timing_reset(); ops.timing_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    ops.pkm_topk_bwd(q, K1, K2, idx, w, dw, dK1, dK2)
e1.record(); torch.cuda.synchronize(); ops.timing_enable(False)
print(f"pkm_topk_bwd T={T} S={S}: {e0.elapsed_time(e1) / 5:.4f} ms  per kernel:",
      {n: round(v[1] / 5, 4) for n, v in sorted(ops.timing_report().items(), key=lambda kv: -kv[1][1])})
