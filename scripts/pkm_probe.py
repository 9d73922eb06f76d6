"""One pkm_topk call at C2 per-head shapes (probe for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2412_09764_b200 import ops
from synthetic import gen
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
H, Dk, k = 4, 1024, 32
q = torch.empty((T, H, Dk), dtype=torch.bfloat16, device="cuda")
K1 = torch.empty((H, S, Dk // 2), dtype=torch.bfloat16, device="cuda")
K2 = torch.empty_like(K1)
ops.synth_fill(q, 0, gen.TAGS["q"])
ops.synth_fill(K1, 0, gen.TAGS["K1"], scale=gen.scale_for("K1", Dk=Dk))
ops.synth_fill(K2, 0, gen.TAGS["K2"], scale=gen.scale_for("K2", Dk=Dk))
for _ in range(3):
    idx, w = ops.pkm_topk(q, K1, K2, k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    idx, w = ops.pkm_topk(q, K1, K2, k)
e1.record()
torch.cuda.synchronize()
print(f"pkm_topk T={T} S={S}: {e0.elapsed_time(e1) / 10:.4f} ms")
ops.timing_reset()
ops.timing_enable(True)
for _ in range(5):
    ops.pkm_topk(q, K1, K2, k)
torch.cuda.synchronize()
ops.timing_enable(False)
print("  per kernel (ms):", {n: round(v[1] / v[0], 4) for n, v in ops.timing_report().items()})
