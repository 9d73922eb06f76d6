"""EmbeddingBag backward strategy comparison on B200 (§3.1.4, P:176;
SURVEY f3): "atomics", "lock", and the sorted "reverse_indices" (this
library's production path) over value dims and index distributions.
Value gradient only (dw is common to all strategies).  Prints one JSON line
per case and a summary; CUDA-event timing, median of reps."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_09764_b200 import ops  # noqa: E402
from synthetic import gen, streams  # noqa: E402

N, T, B = 1 << 20, 16384, 128


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    dvs = [int(x) for x in os.environ.get("DVS", "64,128,256,512,1024,2048,4096").split(",")]
    profiles = os.environ.get("PROFILES", "uniform,zipf1.1,collide50").split(",")
    out = []
    for prof in profiles:
        if prof == "uniform":
            idx = streams.uniform_indices(0, T, B, N)
        elif prof.startswith("zipf"):
            idx = streams.zipf_indices(0, T, B, N, float(prof[4:]))
        else:
            idx = streams.collision_indices(0, T, B, N, int(prof[7:]))
        w = streams.softmax_free_weights(0, T, B)
        di, dw_ = torch.from_numpy(idx).cuda(), torch.from_numpy(w).cuda()
        U = int(np.unique(idx).size)
        for dv in dvs:
            dy = torch.empty((T, dv), dtype=torch.bfloat16, device="cuda")
            ops.synth_fill(dy, 0, gen.TAGS["dout"])
            dense = torch.zeros((N, dv), dtype=torch.float32, device="cuda")
            t_memset = timeit(lambda: dense.zero_())
            t_atom = timeit(lambda: ops.embbag_bwd_atomics(N, di, dw_, dy, dense))
            t_lock = timeit(lambda: ops.embbag_bwd_lock(N, di, dw_, dy, dense), reps=3)
            t_rev = timeit(lambda: ops.embbag_bwd_dv_only(N, di, dw_, dy, sync=False))
            rec = dict(profile=prof, dv=dv, U_over_P=U / idx.size, ms_atomics=t_atom, ms_lock=t_lock,
                       ms_reverse_indices=t_rev, ms_dense_zero=t_memset,
                       fastest=min(("atomics", t_atom), ("lock", t_lock),
                                   ("reverse_indices", t_rev), key=lambda x: x[1])[0])
            print(json.dumps(rec), flush=True)
            out.append(rec)
            del dense, dy
            torch.cuda.empty_cache()
    print("SUMMARY", json.dumps({f"{r['profile']}/{r['dv']}": r["fastest"] for r in out}))


if __name__ == "__main__":
    main()
