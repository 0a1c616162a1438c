"""Batch-sharded multi-GPU driver (one process per GPU, torch.distributed).

Convolution is independent per image, so the forward pass partitions the
minibatch N into contiguous per-rank shards, replicates the filters (each rank
transforms g itself: recomputing U is cheaper than broadcasting it over
NVLink), and needs NO collective.  The only optional exchange is
a verification gather of the outputs (NCCL all_gather over NVLink/NVSwitch).
"""
from __future__ import annotations

from typing import Optional, Tuple

from .layer import LayerConfig


def shard_bounds(N: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced split of N images: (start, count) for `rank`.
    The first N % world ranks take one extra image."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if N < 0:
        raise ValueError("N must be >= 0")
    base, extra = divmod(N, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def local_config(cfg: LayerConfig, world: int, rank: int) -> Optional[LayerConfig]:
    """This rank's layer shape, or None if the rank holds no images."""
    _, n = shard_bounds(cfg.N, world, rank)
    return cfg.with_batch(n) if n > 0 else None


class ShardedForward:
    """Per-rank forward of one layer over its batch shard (device tensors)."""

    def __init__(self, cfg: LayerConfig, m: int, prec: str = "fp32", world: int = 1,
                 rank: int = 0, workspace_limit: int = 0) -> None:
        from .engine import WinogradPlan
        self.global_cfg = cfg
        self.world, self.rank = world, rank
        self.start, self.count = shard_bounds(cfg.N, world, rank)
        self.cfg = local_config(cfg, world, rank)
        self.plan = WinogradPlan(self.cfg, m, prec, workspace_limit) if self.cfg else None
        self.U = None

    def set_filters(self, g, stream=None) -> None:
        """Replicated filters: every rank transforms its own copy (no broadcast)."""
        if self.plan is not None:
            self.U = self.plan.filter_transform(g, stream=stream)

    def forward(self, d_local, y_local=None, workspace=None, stream=None, g=None):
        """This rank's shard of the layer.  FX (the transformed filters from
        set_filters) by default; pass ``g`` for the non-FX forward, which
        transforms the replicated filters inside the call."""
        if self.plan is None:
            return None
        if g is None and self.U is None:
            raise ValueError("call set_filters() first (or pass g)")
        if g is not None:
            return self.plan.forward(d_local, y=y_local, g=g, workspace=workspace, stream=stream)
        return self.plan.forward(d_local, y=y_local, U=self.U, workspace=workspace, stream=stream)

    def local_slice(self, d_global):
        """This rank's contiguous images of a global batch tensor."""
        return d_global[self.start:self.start + self.count]


def shard_bounds_native(N: int, world: int, rank: int) -> Tuple[int, int]:
    """shard_bounds through the C ABI (wino_shard_bounds; host-only)."""
    import ctypes
    from . import _lib
    start, count = ctypes.c_int(), ctypes.c_int()
    _lib.check(_lib.lib.wino_shard_bounds(N, world, rank, ctypes.byref(start),
                                          ctypes.byref(count)), "wino_shard_bounds")
    return start.value, count.value


class DeviceShardedForward:
    """One host thread driving several devices through ``wino_forward_sharded``
    (the C-ABI multi-GPU entry point): shard s = the images
    ``shard_bounds(N, len(devices), s)`` on ``devices[s]`` (devices may repeat),
    filters replicated, no collective.  The torch.distributed driver
    (one process per GPU) is ``ShardedForward``."""

    def __init__(self, cfg: LayerConfig, m: int, prec: str = "fp32", devices=(0,),
                 workspace_limit: int = 0) -> None:
        import ctypes
        import torch
        from . import _lib
        from .engine import WinogradPlan
        self.cfg, self.devices = cfg, [int(x) for x in devices]
        n = len(self.devices)
        if n < 1:
            raise ValueError("need at least one device")
        self.plan = WinogradPlan(cfg, m, prec, workspace_limit)
        self.bounds = [shard_bounds(cfg.N, n, s) for s in range(n)]
        self.U = None
        self._ws = []
        for s, dev in enumerate(self.devices):
            b = ctypes.c_size_t()
            _lib.check(_lib.lib.wino_shard_workspace(self.plan._h, n, s, 1, ctypes.byref(b)),
                       "wino_shard_workspace")
            self._ws.append(torch.empty(max(int(b.value), 1), dtype=torch.uint8,
                                        device=f"cuda:{dev}"))

    def set_filters(self, g) -> None:
        """Replicated filters: U transformed on every shard's device, on that
        device's current stream (the stream forward() enqueues on)."""
        import torch
        self.U = []
        for dev in self.devices:
            with torch.cuda.device(dev):
                self.U.append(self.plan.filter_transform(
                    g.to(device=f"cuda:{dev}", dtype=self.plan.data_dtype).contiguous(),
                    stream=torch.cuda.current_stream(dev)))

    def forward(self, d_shards, y_shards=None, g=None):
        """d_shards[s]: (count_s, C, H, W) on devices[s] -> list of y shards.
        FX with the U of set_filters, or pass ``g`` (any device) to transform the
        filters inside the call.  Enqueued on each device's current stream."""
        import ctypes
        import torch
        from . import _lib
        c, n = self.cfg, len(self.devices)
        if len(d_shards) != n:
            raise ValueError(f"expected {n} input shards, got {len(d_shards)}")
        if g is None and self.U is None:
            raise ValueError("call set_filters() first (or pass g)")
        dt = self.plan.data_dtype
        ys, gs = [], []
        for s, dev in enumerate(self.devices):
            cnt = self.bounds[s][1]
            x = d_shards[s]
            if (not isinstance(x, torch.Tensor) or x.device != torch.device("cuda", dev)
                    or tuple(x.shape) != (cnt, c.C, c.H, c.W) or x.dtype != dt
                    or not x.is_contiguous()):
                raise ValueError(f"shard {s}: expected contiguous {dt} ({cnt}, {c.C}, {c.H}, "
                                 f"{c.W}) on cuda:{dev}")
            y = (y_shards[s] if y_shards is not None else
                 torch.empty((cnt, c.K, c.out_h, c.out_w), dtype=dt, device=f"cuda:{dev}"))
            if (tuple(y.shape) != (cnt, c.K, c.out_h, c.out_w) or y.dtype != dt
                    or y.device != x.device or not y.is_contiguous()):
                raise ValueError(f"shard {s}: bad output tensor")
            ys.append(y)
            if g is not None:
                gs.append(g.to(device=f"cuda:{dev}", dtype=dt).contiguous())
        vpa = ctypes.c_void_p * n
        ptrs = lambda xs: vpa(*[x.data_ptr() if x is not None and x.numel() else None
                                for x in xs])
        streams = vpa(*[torch.cuda.current_stream(dev).cuda_stream for dev in self.devices])
        wsb = (ctypes.c_size_t * n)(*[w.numel() for w in self._ws])
        _lib.check(_lib.lib.wino_forward_sharded(
            self.plan._h, n, (ctypes.c_int * n)(*self.devices), ptrs(d_shards),
            ptrs(self.U) if g is None else None, ptrs(gs) if g is not None else None,
            ptrs(ys), ptrs(self._ws), wsb, streams), "wino_forward_sharded")
        return ys


def gather_outputs(y_local, cfg: LayerConfig, group=None):
    """Optional verification gather of all shards to every rank (all_gather).
    Not part of the forward pass."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = [shard_bounds(cfg.N, world, r)[1] for r in range(world)]
    per = (cfg.K, cfg.out_h, cfg.out_w)
    mx = max(counts)
    buf = torch.zeros((mx, *per), dtype=y_local.dtype, device=y_local.device)
    buf[: y_local.shape[0]] = y_local
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return torch.cat([o[:c] for o, c in zip(outs, counts)], dim=0)
