"""CUDA-graph capture of the memory-layer step (paper_2412_09764_b200/graph.py):
a replay equals the eager step bit for bit (the kernels are deterministic), on
the captured inputs and again after new data is copied into the static input
tensors.  Numerics of the step against the oracle: test_gpu_parity.py."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _inputs(seed, T, D, dv, H, S, Dk, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    bf = torch.bfloat16

    def r(*shape, scale=1.0):
        return (torch.randn(*shape, generator=g, device=dev) * scale).to(bf)
    return dict(x=r(T, D), q=r(T, H, Dk), dout=r(T, D),
                K1=r(H, S, Dk // 2, scale=Dk ** -0.5), K2=r(H, S, Dk // 2, scale=Dk ** -0.5),
                V=r(S * S, dv), W1=r(D, dv, scale=D ** -0.5), W2=r(dv, D, scale=dv ** -0.5))


def _eager(t, k, qk_norm):
    from paper_2412_09764_b200 import ops
    dK1 = torch.zeros(t["K1"].shape, dtype=torch.float32, device=t["q"].device)
    dK2 = torch.zeros_like(dK1)
    out, saved = ops.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"],
                                      k, qk_norm=qk_norm)
    g = ops.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"],
                             saved, dK1=dK1, dK2=dK2)
    return out, g


def _assert_same(a, b):
    (oa, ga), (ob, gb) = a, b
    torch.cuda.synchronize()
    assert torch.equal(oa, ob)
    for name in ("dq", "dK1", "dK2", "dx", "dW1", "dW2"):
        assert torch.equal(getattr(ga, name), getattr(gb, name)), name
    U = int(ga.U.item())
    assert U == int(gb.U.item()) and U > 0
    assert torch.equal(ga.rows[:U], gb.rows[:U])
    assert torch.equal(ga.dV[:U], gb.dV[:U])


@pytest.mark.parametrize("qk_norm", [False, True])
def test_graph_replay_bit_identical(qk_norm):
    from paper_2412_09764_b200.graph import MemoryLayerStepGraph
    dev = torch.device("cuda", 0)
    T, D, dv, H, S, Dk, k = 300, 256, 256, 2, 64, 128, 8   # ragged T
    t = _inputs(1, T, D, dv, H, S, Dk, dev)
    gr = MemoryLayerStepGraph(t["x"], t["q"], t["dout"], t["K1"], t["K2"], t["V"], t["W1"],
                              t["W2"], k, qk_norm=qk_norm)
    _assert_same(gr.replay(), _eager(t, k, qk_norm))
    # new data through the static inputs
    t2 = _inputs(2, T, D, dv, H, S, Dk, dev)
    for name in ("x", "q", "dout"):
        t[name].copy_(t2[name])
    _assert_same(gr.replay(), _eager(t, k, qk_norm))
    # replays are repeatable (dK accumulators are zeroed inside the graph)
    first = [x.clone() for x in (gr.out, gr.grads.dK1, gr.grads.dW1)]
    gr.replay()
    torch.cuda.synchronize()
    for a, b in zip(first, (gr.out, gr.grads.dK1, gr.grads.dW1)):
        assert torch.equal(a, b)
