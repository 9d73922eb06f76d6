"""CUDA-graph capture of one memory-layer training step (forward + backward).

    g = MemoryLayerStepGraph(x, q, dout, K1, K2, V, W1, W2, k)
    x.copy_(next_x); q.copy_(next_q); dout.copy_(next_dout)   # static inputs
    out, grads = g.replay()

Everything the step launches (product-key scoring and top-k, softmax, the bag
forward with the fused gate, the gate GEMMs, the sorted inverse index map on
the library's side stream, the segmented backward, the key/query gradients) is
captured once; a replay re-issues the whole DAG with one launch.  The library's
side streams fork from and join the capturing stream through events, so they
are part of the graph.  Replays are bit-identical to the eager step (the path
is deterministic; tests/test_gpu_graph.py).

Measured on one B200 (scripts/graph_probe.py, C2 shapes with T tokens): the
replay saves the host launch overhead of ~40 launches, 1.39x at T = 256 and
1.07x at T = 1024; from T = 4096 up the GPU is never starved and graph and
eager steps take the same time, so bench.py times the eager step by default.

Shapes, dtypes and tensor addresses are fixed at capture: feed new data by
copying into the static input tensors passed here.  dK1/dK2 are zeroed inside
the graph (each replay returns this step's key gradients).
"""
import torch

from . import ops


class MemoryLayerStepGraph:
    def __init__(self, x, q, dout, K1, K2, V, W1, W2, k, qk_norm=False, warmup=3):
        self.x, self.q, self.dout = x, q, dout
        self.K1, self.K2, self.V, self.W1, self.W2 = K1, K2, V, W1, W2
        self.k, self.qk_norm = k, qk_norm
        dev = q.device
        self.dK1 = torch.zeros(K1.shape, dtype=torch.float32, device=dev)
        self.dK2 = torch.zeros(K2.shape, dtype=torch.float32, device=dev)
        self._bufs = {}
        # warm-up and capture on one private stream: the library creates its
        # side streams and tunes its GEMMs (first call, host-synchronising)
        # here, outside the capture
        self.stream = torch.cuda.Stream(device=dev)
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(self.stream):
            for _ in range(max(1, warmup)):
                self._step()
        torch.cuda.current_stream(dev).wait_stream(self.stream)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self.out, self.grads = self._step()

    def _step(self):
        self.dK1.zero_()
        self.dK2.zero_()
        out, saved = ops.memory_layer_fwd(self.x, self.q, self.K1, self.K2, self.V, self.W1,
                                          self.W2, self.k, qk_norm=self.qk_norm, keep_state=True)
        g = ops.memory_layer_bwd(self.dout, self.x, self.q, self.K1, self.K2, self.V, self.W1,
                                 self.W2, saved, dK1=self.dK1, dK2=self.dK2, bufs=self._bufs)
        return out, g

    def replay(self):
        """Enqueue one captured step on the current stream; returns the static
        outputs (valid once the stream reaches this point)."""
        self.graph.replay()
        return self.out, self.grads
