"""The autograd wrapper (paper_2412_09764_b200/layer.py) is wiring only: its
parameter gradients equal the C-ABI backward's outputs bit for bit (the
kernels are deterministic), sparse and dense value gradients agree, and the
module runs on [batch, seq, D] inputs.  Numerics of the layer itself against
the oracle are covered by test_gpu_parity.py."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


@pytest.mark.parametrize("dense", [False, True])
def test_memory_layer_module_grads_match_cabi(dense):
    from paper_2412_09764_b200 import ops
    from paper_2412_09764_b200.layer import MemoryLayer
    torch.manual_seed(0)
    dev = torch.device("cuda", 0)
    layer = MemoryLayer(D=256, dv=256, H=2, S=64, Dk=128, k=8, dense_value_grad=dense, device=dev)
    x = torch.randn(2, 40, 256, device=dev, dtype=torch.bfloat16, requires_grad=True)
    y = layer(x)
    assert y.shape == x.shape
    loss = y.float().square().sum()
    loss.backward()
    # the same step straight through the C ABI
    x2 = x.detach().reshape(-1, 256)
    q = layer.query(x2).detach().reshape(-1, 2, 128).contiguous()
    out, saved = ops.memory_layer_fwd(x2, q, layer.K1.detach(), layer.K2.detach(), layer.V.detach(),
                                      layer.W1.detach(), layer.W2.detach(), 8)
    assert torch.equal(out, y.detach().reshape(-1, 256))
    dout = (2.0 * out.float()).to(out.dtype)
    g = ops.memory_layer_bwd(dout, x2, q, layer.K1.detach(), layer.K2.detach(), layer.V.detach(),
                             layer.W1.detach(), layer.W2.detach(), saved)
    torch.cuda.synchronize()
    assert torch.equal(layer.K1.grad, g.dK1.to(layer.K1.dtype))
    assert torch.equal(layer.K2.grad, g.dK2.to(layer.K2.dtype))
    assert torch.equal(layer.W1.grad, g.dW1.to(layer.W1.dtype))
    assert torch.equal(layer.W2.grad, g.dW2.to(layer.W2.dtype))
    U = int(g.U.item())
    ref = torch.zeros(layer.V.shape, dtype=torch.float32, device=dev)
    ref[g.rows[:U].long()] = g.dV[:U]
    vg = layer.V.grad.to_dense() if layer.V.grad.is_sparse else layer.V.grad
    assert layer.V.grad.is_sparse == (not dense)
    assert torch.equal(vg, ref.to(layer.V.dtype))
    assert x.grad is not None and torch.isfinite(x.grad.float()).all()
