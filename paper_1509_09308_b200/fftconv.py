"""FFT overlap-and-save layer on the GPU: the reference's ``fft`` comparison
algorithm (winoconv/fftconv.py:206-275, paper sec. 4.4).  Not the Winograd
hot path.  Hand-written CUDA kernels (csrc/wino_fft.cu, C ABI
``wino_fft_forward``): direct 8x8 DFTs of the reversed filters and of the
zero-filled input tiles (virtual padding), a complex fp64 batched GEMM over the
Hermitian-unique frequencies, and the real inverse DFT with the clipped
scatter -- all in fp64 like the reference (numpy complex128), the output cast
to the input type.  Counter semantics follow the reference's fast path:
``"cmul" += Q*K*C*P`` and ``"mul" += 3*Q*K*C*P`` (fftconv.py:153-168).
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from .layer import LayerConfig, OpCounter
from .tensors import Precision, Tensor4, precision_of


def fft_forward_layer(d, g, cfg: LayerConfig, tile: int = 8,
                      counter: Optional[OpCounter] = None, fast: bool = True) -> Tensor4:
    """Tiled FFT correlation (fftconv.py:206-275); same ValueErrors.  The GPU
    path implements run_layer's tile (8); other tiles raise ValueError."""
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

    desc = _lib.LayerDesc(cfg.N, cfg.C, cfg.H, cfg.W, cfg.K, cfg.R, cfg.S, cfg.pad)
    ws_bytes = ctypes.c_size_t()
    _lib.check(_lib.lib.wino_fft_workspace(ctypes.byref(desc), tile, ctypes.byref(ws_bytes)),
               "wino_fft_workspace")
    f64 = dp is Precision.FP64
    dt = np.float64 if f64 else np.float32
    d_dev = torch.from_numpy(np.array(d.data, dtype=dt, order="C")).cuda()
    g_dev = torch.from_numpy(np.array(g.data, dtype=np.float64, order="C")).cuda()
    y = torch.empty((cfg.N, cfg.K, cfg.out_h, cfg.out_w),
                    dtype=torch.float64 if f64 else torch.float32, device="cuda")
    ws = torch.empty(ws_bytes.value, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib.wino_fft_forward(
        ctypes.byref(desc), _lib.PREC_FP64 if f64 else _lib.PREC_FP32, tile, d_dev.data_ptr(),
        g_dev.data_ptr(), y.data_ptr(), ws.data_ptr(), ws_bytes.value,
        torch.cuda.current_stream().cuda_stream), "wino_fft_forward")
    if counter is not None:
        a = tile
        gh = -(-cfg.out_h // (a - cfg.R + 1))
        gw = -(-cfg.out_w // (a - cfg.S + 1))
        Q, P = a * (a // 2 + 1), cfg.N * gh * gw
        counter.add("cmul", Q * cfg.K * cfg.C * P)
        counter.add("mul", (3 if fast else 4) * Q * cfg.K * cfg.C * P)
    out = y.cpu().numpy()
    return Tensor4._wrap(out, Precision.FP64 if f64 else Precision.FP32)
