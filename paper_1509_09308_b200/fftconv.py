"""FFT overlap-and-save layer on the GPU: the reference's ``fft`` comparison
algorithm (winoconv/fftconv.py:206-275, paper sec. 4.4).  Not the Winograd
hot path: it uses cuFFT and a complex128 batched GEMM through torch, with the
reference's tiling (alpha = tile, outputs (alpha-R+1) x (alpha-S+1) per tile),
its fp64 transform-space arithmetic and its Hermitian-unique frequency set, so
results agree with the reference to fp64 rounding before the final cast.
Counter semantics follow the reference's fast path: ``"cmul" += Q*K*C*P`` and
``"mul" += 3*Q*K*C*P`` (three real GEMMs, fftconv.py:153-168).
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from .layer import LayerConfig, OpCounter
from .tensors import Precision, Tensor4, precision_of


def fft_forward_layer(d, g, cfg: LayerConfig, tile: int = 8,
                      counter: Optional[OpCounter] = None, fast: bool = True) -> Tensor4:
    """Tiled FFT correlation (fftconv.py:206-275); same ValueErrors."""
    if tile < 1 or tile & (tile - 1):
        raise ValueError(f"tile must be a power of two, got {tile}")
    if tile <= cfg.R - 1 or tile <= cfg.S - 1:
        raise ValueError(f"tile {tile} too small for a {cfg.R}x{cfg.S} filter")
    dp, gp = precision_of(d), precision_of(g)
    if dp != gp:
        raise ValueError(f"mixed precisions: {dp} vs {gp}")
    if tuple(d.shape) != (cfg.N, cfg.C, cfg.H, cfg.W):
        raise ValueError(f"data shape {d.shape} does not match {cfg}")
    if tuple(g.shape) != (cfg.K, cfg.C, cfg.R, cfg.S):
        raise ValueError(f"filter shape {g.shape} does not match {cfg}")
    import torch
    import torch.nn.functional as F

    a = tile
    mh, mw = a - cfg.R + 1, a - cfg.S + 1
    oh, ow = cfg.out_h, cfg.out_w
    gh, gw = -(-oh // mh), -(-ow // mw)
    P = cfg.N * gh * gw
    half = a // 2
    Q = a * (half + 1)
    dev = torch.device("cuda")
    # reversed, zero-padded filters: cyclic convolution realises correlation
    gt = torch.from_numpy(np.array(g.data, dtype=np.float64)).to(dev)
    h = torch.zeros((cfg.K, cfg.C, a, a), dtype=torch.float64, device=dev)
    h[:, :, :cfg.R, :cfg.S] = torch.flip(gt, dims=(2, 3))
    ghat = torch.fft.rfft2(h)                                   # (K, C, a, half+1)
    # zero-filled a x a tiles at (mh*ty - pad, mw*tx - pad)
    dt = torch.from_numpy(np.array(d.data, dtype=np.float64)).to(dev)
    need_h, need_w = mh * (gh - 1) + a, mw * (gw - 1) + a
    dpad = F.pad(dt, (cfg.pad, max(0, need_w - cfg.W - cfg.pad),
                      cfg.pad, max(0, need_h - cfg.H - cfg.pad)))
    tiles = dpad.unfold(2, a, mh).unfold(3, a, mw)[:, :, :gh, :gw]  # (N, C, gh, gw, a, a)
    tiles = tiles.permute(0, 2, 3, 1, 4, 5).reshape(P, cfg.C, a, a)
    dhat = torch.fft.rfft2(tiles)                               # (P, C, a, half+1)
    u = ghat.permute(2, 3, 0, 1).reshape(Q, cfg.K, cfg.C)
    v = dhat.permute(2, 3, 1, 0).reshape(Q, cfg.C, P)
    m = torch.matmul(u, v)                                      # (Q, K, P) complex128
    if counter is not None:
        counter.add("cmul", Q * cfg.K * cfg.C * P)
        counter.add("mul", (3 if fast else 4) * Q * cfg.K * cfg.C * P)
    plane = m.reshape(a, half + 1, cfg.K, P).permute(2, 3, 0, 1)
    y = torch.fft.irfft2(plane, s=(a, a))                       # (K, P, a, a)
    valid = y[:, :, cfg.R - 1:, cfg.S - 1:].reshape(cfg.K, cfg.N, gh, gw, mh, mw)
    full = valid.permute(1, 0, 2, 4, 3, 5).reshape(cfg.N, cfg.K, gh * mh, gw * mw)
    out_dt = torch.float64 if dp is Precision.FP64 else torch.float32
    out = full[:, :, :oh, :ow].to(out_dt).contiguous().cpu().numpy()
    return Tensor4._wrap(out, Precision.FP64 if dp is Precision.FP64 else Precision.FP32)
