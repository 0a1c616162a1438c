"""The chained VGG-E stack (network.VGGEStack): 16 Winograd conv layers with
ReLU and 2x2 max-pool between blocks, against the same network in fp64 with
torch's direct convolution."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fuse", [True, False])
@pytest.mark.parametrize("m,prec,tol", [(2, "fp32", 1e-4), (4, "fp32", 1e-3),
                                        (4, "fp16", 5e-2)])
def test_vgg_e_stack_matches_fp64_network(m, prec, tol, fuse):
    import torch
    from paper_1509_09308_b200.network import VGGEStack
    net = VGGEStack(2, m, prec, seed=3, fuse_act=fuse)
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


def test_fused_act_stack_bitwise_equal_to_separate_pass():
    """ReLU / max-pool fused into the output transform give the separate
    wino_relu_pool pass's result bit for bit (same conv values, same max)."""
    import torch
    from paper_1509_09308_b200.network import VGGEStack
    for m in (2, 4):
        a = VGGEStack(1, m, "fp32", seed=4, fuse_act=True)
        b = VGGEStack(1, m, "fp32", seed=4, fuse_act=False)
        x = torch.rand(a.in_shape, device="cuda") * 2 - 1
        ya, yb = a.forward(x), b.forward(x)
        torch.cuda.synchronize()
        assert torch.equal(ya, yb), m


@pytest.mark.parametrize("m", [2, 4])
@pytest.mark.parametrize("N,C,H,K", [(2, 3, 30, 16),     # small-C whole-layer kernel
                                     (1, 64, 28, 96),    # TMA output transform
                                     (1, 256, 14, 256),  # split-C / per-thread output
                                     (3, 40, 22, 72)])   # F4 edge tiles (22 % 4 == 2)
@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_forward_act_matches_torch_epilogue(m, N, C, H, K, prec):
    """wino_forward_act: relu(y) and maxpool2x2(relu(y)) equal torch's ops on the
    plain forward's output, bitwise."""
    import torch
    import torch.nn.functional as F
    import paper_1509_09308_b200 as wb
    cfg = wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
    plan = wb.WinogradPlan(cfg, m, prec)
    d = torch.rand((N, C, H, H), device="cuda") * 2 - 1
    g = torch.rand((K, C, 3, 3), device="cuda") * 2 - 1
    y = plan.forward(d, g=g)
    r = plan.forward(d, g=g, act="relu")
    p = plan.forward(d, g=g, act="relu_pool")
    torch.cuda.synchronize()
    assert torch.equal(r, torch.relu(y))
    assert p.shape == (N, K, H // 2, H // 2)
    assert torch.equal(p, F.max_pool2d(torch.relu(y), 2))


def test_forward_act_errors(monkeypatch):
    import torch
    import paper_1509_09308_b200 as wb
    d = torch.rand((1, 16, 9, 9), device="cuda")
    g = torch.rand((8, 16, 3, 3), device="cuda")
    plan = wb.WinogradPlan(wb.LayerConfig(N=1, C=16, H=9, W=9, K=8, pad=1), 2, "fp32")
    with pytest.raises(ValueError):  # odd output: no 2x2 pooling
        plan.forward(d, g=g, y=torch.empty((1, 8, 4, 4), device="cuda"), act="relu_pool")
    with pytest.raises(ValueError):
        plan.forward(d, g=g, act="gelu")
    monkeypatch.setenv("WINO_PATH", "fused")
    fused = wb.WinogradPlan(wb.LayerConfig(N=1, C=16, H=10, W=10, K=8, pad=1), 2, "fp32")
    with pytest.raises(ValueError):  # the epilogue runs on the staged path only
        fused.forward(torch.rand((1, 16, 10, 10), device="cuda"), g=g, act="relu")


def test_fx_stack_equals_non_fx():
    """fx=True transforms the filters once (FilterCache semantics); the forward
    with the cached U is bitwise the non-FX forward."""
    import torch
    from paper_1509_09308_b200.network import VGGEStack
    a = VGGEStack(1, 4, "bf16", seed=6, fx=True)
    b = VGGEStack(1, 4, "bf16", seed=6, fx=False)
    x = torch.rand(a.in_shape, device="cuda") * 2 - 1
    ya, yb = a.forward(x), b.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)
