"""wino_forward_sharded: one host thread, several shards through the C ABI
(SURVEY.md §8(b) / §8(e)).  The box has one GPU, so the shards share cuda:0;
the per-device plumbing (cudaSetDevice per shard, per-device side streams) is
the same code path as on a multi-GPU node."""
import pytest
import torch

from paper_1509_09308_b200 import LayerConfig
from paper_1509_09308_b200.engine import WinogradPlan
from paper_1509_09308_b200.sharding import DeviceShardedForward

pytestmark = pytest.mark.gpu


def _inputs(cfg, seed):
    gen = torch.Generator(device="cpu").manual_seed(seed)
    d = (torch.rand((cfg.N, cfg.C, cfg.H, cfg.W), generator=gen) * 2 - 1).cuda()
    g = (torch.rand((cfg.K, cfg.C, 3, 3), generator=gen) * 2 - 1).cuda()
    return d, g


@pytest.mark.parametrize("m,prec,N,C,H,K,shards", [
    (2, "fp32", 5, 64, 28, 64, 3),     # ragged: 2 / 2 / 1 images
    (4, "bf16", 8, 128, 56, 128, 4),
    (4, "fp16", 3, 256, 14, 512, 2),   # K > P on every shard
    (2, "fp32", 2, 3, 32, 64, 4),      # small-C kernel; two shards without images
    (4, "tf32", 64, 512, 14, 512, 8),  # config 4's conv5 split, 8 images per shard
    (4, "fp64", 3, 16, 12, 8, 2),      # fp64 data on the CUDA-core GEMM
])
def test_sharded_equals_per_shard_plans(m, prec, N, C, H, K, shards):
    """Each shard is bitwise the forward of a plan built for its own batch, FX
    and non-FX, and the gathered output matches the direct convolution."""
    cfg = LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
    d, g = _inputs(cfg, 7)
    if prec == "fp64":
        d, g = d.double(), g.double()
    sf = DeviceShardedForward(cfg, m, prec, devices=[0] * shards)
    parts = [d[s:s + c].contiguous() for s, c in sf.bounds]
    sf.set_filters(g)
    ys = sf.forward(parts)
    ys_g = sf.forward(parts, g=g)
    torch.cuda.synchronize()
    for (s, c), y, yg, x in zip(sf.bounds, ys, ys_g, parts):
        assert y.shape == (c, K, H, H)
        if c == 0:
            continue
        ref = WinogradPlan(cfg.with_batch(c), m, prec).forward(x, g=g)
        torch.cuda.synchronize()
        assert torch.equal(y, ref), (s, c)
        assert torch.equal(yg, ref), (s, c)
    y = torch.cat(ys)
    exact = torch.nn.functional.conv2d(d.double(), g.double(), padding=1)
    rel = ((y.double() - exact).abs().max() / exact.abs().max()).item()
    tol = {("fp32", 2): 5e-5, ("tf32", 4): 4e-2, ("bf16", 4): 1.5e-1, ("fp16", 4): 2.5e-2,
           ("fp64", 4): 1e-12}
    assert rel <= tol[(prec, m)], rel  # test_gpu_parity.REL_TOL; fp32 within the 5e-4 gate


def test_sharded_errors_name_the_shard():
    cfg = LayerConfig(N=4, C=16, H=8, W=8, K=16, pad=1)
    d, g = _inputs(cfg, 1)
    sf = DeviceShardedForward(cfg, 2, "fp32", devices=[0, 0])
    parts = [d[:2].contiguous(), d[2:].contiguous()]
    with pytest.raises(ValueError):
        sf.forward(parts)  # no filters yet
    with pytest.raises(ValueError):
        sf.forward(parts[:1], g=g)
    with pytest.raises(ValueError):
        sf.forward([parts[0], d[:3].contiguous()], g=g)
    sf._ws[1] = sf._ws[1][:16]  # undersized workspace on shard 1
    with pytest.raises(ValueError, match="shard 1"):
        sf.forward(parts, g=g)
