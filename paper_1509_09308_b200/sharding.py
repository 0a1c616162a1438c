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
