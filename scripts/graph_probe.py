"""CUDA-graph capture of one memory-layer step (fwd + bwd) through the public API.

For each token count T (C2 shapes otherwise: N = 1024^2, dv = D = 2048, 4 heads,
k = 32, bf16): run the step eagerly, capture the same step into a
torch.cuda.CUDAGraph (the library's side streams fork from / join the capturing
stream by events, so they are captured too), replay it, check that the replayed
outputs equal the eager ones bit for bit, and time both with CUDA events.
Prints one JSON line per T.  GPU only; not part of the bench contract.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2412_09764_b200 import ops  # noqa: E402


def flat(out, g):
    ts = [out]
    for v in (g.values() if isinstance(g, dict) else vars(g).values()):
        if torch.is_tensor(v):
            ts.append(v)
    return ts


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    steps = int(os.environ.get("GP_STEPS", "50"))
    base = dict(bench.CONFIGS["c2"])
    t_all = None
    for T in [int(x) for x in os.environ.get("GP_T", "256,1024,4096,16384").split(",")]:
        cfg = dict(base, T=T)
        t = bench.make_inputs(cfg, dev, 1, 0, ops, torch)
        if t_all is not None:
            t["V"] = t_all  # reuse the 4 GiB table
        t_all = t["V"]
        dK1 = torch.zeros(t["K1"].shape, dtype=torch.float32, device=dev)
        dK2 = torch.zeros(t["K2"].shape, dtype=torch.float32, device=dev)
        bufs = {}

        def step():
            dK1.zero_()
            dK2.zero_()
            out, saved = ops.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"],
                                              t["W1"], t["W2"], cfg["k"])
            g = ops.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"],
                                     t["W1"], t["W2"], saved, dK1=dK1, dK2=dK2, bufs=bufs)
            return out, g

        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(5):
                out, g = step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        eager = [x.clone() for x in flat(out, g)] + [dK1.clone(), dK2.clone()]

        def timed(fn):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / steps

        ms_eager = timed(step)

        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):  # aux streams already exist for s
            gout, gg = step()
        graph.replay()
        torch.cuda.synchronize()
        replayed = [x.clone() for x in flat(gout, gg)] + [dK1.clone(), dK2.clone()]
        same = len(eager) == len(replayed) and all(
            a.shape == b.shape and torch.equal(a, b) for a, b in zip(eager, replayed))
        ms_graph = timed(graph.replay)
        print(json.dumps(dict(T=T, ms_eager=round(ms_eager, 4), ms_graph=round(ms_graph, 4),
                              speedup=round(ms_eager / ms_graph, 3),
                              tok_s_eager=round(T / ms_eager * 1e3),
                              tok_s_graph=round(T / ms_graph * 1e3),
                              bit_identical=bool(same), tensors=len(eager))), flush=True)
        del graph, gout, gg, out, g, eager, replayed


if __name__ == "__main__":
    main()
