"""The chained VGG-E stack (network.VGGEStack): 16 Winograd conv layers with
ReLU and 2x2 max-pool between blocks, against the same network in fp64 with
torch's direct convolution."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,prec,tol", [(2, "fp32", 1e-4), (4, "fp32", 1e-3),
                                        (4, "fp16", 5e-2)])
def test_vgg_e_stack_matches_fp64_network(m, prec, tol):
    import torch
    from paper_1509_09308_b200.network import VGGEStack
    net = VGGEStack(2, m, prec, seed=3)
    x = torch.rand(net.in_shape, device="cuda") * 2 - 1
    y = net.forward(x)
    torch.cuda.synchronize()
    ref = net.reference(x)
    assert y.shape == ref.shape == (2, 512, 7, 7)
    rel = float((y.double() - ref).abs().max() / ref.abs().max())
    assert rel < tol, rel


def test_relu_pool_kernel():
    import torch
    import torch.nn.functional as F
    from paper_1509_09308_b200 import _lib
    x = torch.randn(2, 3, 10, 14, device="cuda")
    y = torch.empty(2, 3, 5, 7, device="cuda")
    _lib.check(_lib.lib.wino_relu_pool(x.data_ptr(), y.data_ptr(), 2, 3, 10, 14, 1,
                                       torch.cuda.current_stream().cuda_stream))
    z = torch.empty_like(x)
    _lib.check(_lib.lib.wino_relu_pool(x.data_ptr(), z.data_ptr(), 2, 3, 10, 14, 0,
                                       torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert torch.equal(y, torch.relu(F.max_pool2d(x, 2)))
    assert torch.equal(z, torch.relu(x))
    with pytest.raises(ValueError):
        _lib.check(_lib.lib.wino_relu_pool(x.data_ptr(), y.data_ptr(), 2, 3, 9, 14, 1, None))
