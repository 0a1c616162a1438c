"""Chained VGG-E conv stack on the Winograd path.

The reference benchmarks every VGG-E layer on its own input (cmd_bench,
commands.py:136-178; suites.py:68-78).  This chains them the way network E
runs: the 16 3x3 conv layers in order, a ReLU after each
and a 2x2 / stride-2 max-pool closing each block (224 -> 112 -> 56 -> 28 -> 14
-> 7), so layer i's output is layer i+1's input.  Each conv is one
``WinogradPlan`` forward (the drop-in path); the ReLU / pool glue is
``wino_relu_pool``.  Weights are U[-1, 1) scaled by sqrt(3 / (9 C)) (unit
output variance per layer, so activations stay O(1) through 16 layers).
Activations are fp32 NCHW, the reference's data type.

The ReLU and the pool are fused into each conv's output transform
(``wino_forward_act``): the conv writes relu(y), or the pooled relu(y), so no
separate pass re-reads the activations (``fuse_act=False`` keeps the separate
``wino_relu_pool`` pass).
"""
from __future__ import annotations

import ctypes
from typing import List, Optional

from . import _lib
from .engine import WinogradPlan, _stream_handle
from .layer import LayerConfig, gflops_direct
from .suites import VGG_E_ROWS


def vgg_e_layers():
    """(label, C, H, K, pool_after) for the 16 conv layers of network E."""
    out = []
    for (lbl, C, H, K, depth) in VGG_E_ROWS:
        block, _, idx = lbl.partition(".")
        for j in range(depth):
            cin = C if j == 0 else K
            out.append((f"{block}.{int(idx or 1) + j}", cin, H, K, False))
    # a block ends where the next layer's resolution halves, and after the last
    for i, (name, C, H, K, _) in enumerate(out):
        last = i + 1 == len(out) or out[i + 1][2] != H
        out[i] = (name, C, H, K, last)
    return out


class VGGEStack:
    """One network-E conv stack at batch N on the current CUDA device."""

    def __init__(self, N: int, m: int = 2, prec: str = "fp32", seed: int = 0,
                 workspace_limit: int = 0, fuse_act: bool = True, fx: bool = False) -> None:
        import torch
        self.N, self.m, self.prec = N, m, prec
        self.fuse_act = fuse_act
        self.fx = fx  # FX: filters transformed once here, like the reference's FilterCache
        self.layers = []
        gen = torch.Generator(device="cpu").manual_seed(seed)
        act_max = N * 3 * 224 * 224
        ws_max = 0
        for (name, C, H, K, pool) in vgg_e_layers():
            cfg = LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
            plan = WinogradPlan(cfg, m, prec, workspace_limit)
            g = ((torch.rand((K, C, 3, 3), generator=gen) * 2 - 1)
                 * (3.0 / (9 * C)) ** 0.5).cuda()
            self.layers.append((name, cfg, plan, g, pool))
            act_max = max(act_max, N * K * H * H)
            ws_max = max(ws_max, plan.workspace_bytes)
        self.gflop = sum(gflops_direct(c) for (_, c, _, _, _) in self.layers)
        # ping-pong activations (ReLU / pool outputs) + the conv output scratch:
        # a layer never writes the buffer it reads
        self._a = torch.empty(act_max, dtype=torch.float32, device="cuda")
        self._b = torch.empty(act_max, dtype=torch.float32, device="cuda")
        self._c = torch.empty(act_max, dtype=torch.float32, device="cuda")
        self._ws = torch.empty(ws_max, dtype=torch.uint8, device="cuda")
        self._U = [plan.filter_transform(g) if fx else None for (_, _, plan, g, _) in self.layers]
        last = self.layers[-1][1]
        self.out_shape = (N, last.K, last.H // 2, last.W // 2)

    @property
    def in_shape(self):
        return (self.N, 3, 224, 224)

    def launches(self) -> int:
        return sum(p.info["launches_per_forward"]
                   + (0 if (self.fx or p.info["combined_transforms"]) else 1)
                   + (0 if self.fuse_act else 1) for (_, _, p, _, _) in self.layers)

    def forward(self, x, out=None, stream=None):
        """x: (N, 3, 224, 224) fp32 CUDA tensor -> (N, 512, 7, 7)."""
        import torch
        if tuple(x.shape) != self.in_shape or x.dtype != torch.float32 or not x.is_cuda:
            raise ValueError(f"input must be a CUDA fp32 tensor of shape {self.in_shape}")
        sh = _stream_handle(stream)
        cur = x.contiguous()
        bufs = (self._a, self._b)
        for i, (name, cfg, plan, g, pool) in enumerate(self.layers):
            oh = cfg.H // 2 if pool else cfg.H
            last = i + 1 == len(self.layers)
            nxt = (out if (last and out is not None) else
                   bufs[(i + 1) % 2][: cfg.N * cfg.K * oh * oh].view(cfg.N, cfg.K, oh, oh))
            wg = dict(U=self._U[i]) if self.fx else dict(g=g)
            if self.fuse_act:  # relu (+ pool) in the output transform's stores
                plan.forward(cur, y=nxt, workspace=self._ws, stream=stream,
                             act="relu_pool" if pool else "relu", **wg)
            else:
                y = self._c[: cfg.N * cfg.K * cfg.H * cfg.W].view(cfg.N, cfg.K, cfg.H, cfg.W)
                plan.forward(cur, y=y, workspace=self._ws, stream=stream, **wg)
                _lib.check(_lib.lib.wino_relu_pool(y.data_ptr(), nxt.data_ptr(), cfg.N, cfg.K,
                                                   cfg.H, cfg.W, 1 if pool else 0, sh),
                           "relu_pool")
            cur = nxt
        return cur

    def reference(self, x):
        """The same stack in fp64 with torch's direct convolution (test oracle)."""
        import torch
        import torch.nn.functional as F
        cur = x.double()
        for (name, cfg, plan, g, pool) in self.layers:
            cur = torch.relu(F.conv2d(cur, g.double(), padding=1))
            if pool:
                cur = F.max_pool2d(cur, 2)
        return cur
