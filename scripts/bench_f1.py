"""SURVEY f1 measurement at C2 scale: backward of 3 memory layers sharing one
value pool (one pooled sort+reduction vs three separate calls) and the
sparse Adam step on the compact gradient.  CUDA-event medians."""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_09764_b200 import ops  # noqa: E402
from synthetic import gen  # noqa: E402

N, dv, T, H, k, L = 1 << 20, 2048, 16384, 4, 32, 3
B = H * k


def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))


V = torch.empty((N, dv), dtype=torch.bfloat16, device="cuda"); ops.synth_fill(V, 0, gen.TAGS["V"])
K1 = torch.empty((H, 1024, 512), dtype=torch.bfloat16, device="cuda"); ops.synth_fill(K1, 0, 2, scale=gen.scale_for("K1", Dk=1024))
K2 = torch.empty((H, 1024, 512), dtype=torch.bfloat16, device="cuda"); ops.synth_fill(K2, 0, 3, scale=gen.scale_for("K1", Dk=1024))
lay = []
for l in range(L):
    q = torch.empty((T, H, 1024), dtype=torch.bfloat16, device="cuda"); ops.synth_fill(q, l, 1)
    idx, w = ops.pkm_topk(q, K1, K2, k)
    dy = torch.empty((T, dv), dtype=torch.bfloat16, device="cuda"); ops.synth_fill(dy, l, 8)
    lay.append((idx.view(T, B), w.view(T, B), dy))
t_sep = timeit(lambda: [ops.embbag_bwd(V, i, w, d, sync=False) for i, w, d in lay])
t_pool = timeit(lambda: ops.embbag_bwd_pool(V, [i for i, _, _ in lay], [w for _, w, _ in lay], [d for _, _, d in lay]))
rows, dV, U, _ = ops.embbag_bwd_pool(V, [i for i, _, _ in lay], [w for _, w, _ in lay], [d for _, _, d in lay])
u = int(U.item())
m = torch.zeros((N, dv), device="cuda"); v = torch.zeros((N, dv), device="cuda")
st = torch.zeros(N, dtype=torch.int32, device="cuda"); Vm = V.float()
t_adam = timeit(lambda: ops.sparse_adam(V, rows, dV, U, m, v, st, lr=1e-3, V_master=Vm))
adam_bytes = u * dv * (4 + 2 * 4 * 2 + 4 * 2 + 2)   # g read, m/v rw, master rw, bf16 V write
print(json.dumps(dict(layers=L, tokens_per_layer=T, U_pooled=u, P_total=L * T * B,
                      ms_three_separate_backwards=t_sep, ms_pooled_backward=t_pool,
                      ms_sparse_adam=t_adam, sparse_adam_GBs=adam_bytes / t_adam / 1e6)))
