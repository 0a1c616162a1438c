"""Direct correlation on the GPU (C ABI ``wino_direct_forward``): the
reference's ``direct`` / ``direct-fp32`` algorithms and the fp64 oracle of
``cmd_accuracy`` (winoconv/direct.py:82-114).  The CUDA kernel accumulates in
the reference's order (c, then v, then u) with a rounded multiply and a rounded
add, so results are bitwise the reference's.  Not the Winograd hot path.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from .layer import LayerConfig, OpCounter
from .tensors import Precision, Tensor4, precision_of


def _valid_taps(cfg: LayerConfig) -> int:
    """Multiplies the reference counts: N*K*(valid window) per (c, v, u)
    (direct.py:100-113)."""
    oh, ow = cfg.out_h, cfg.out_w
    total = 0
    for v in range(cfg.S):
        co = v - cfg.pad
        ys, ye = max(0, -co), min(ow, cfg.W - co)
        for u in range(cfg.R):
            ro = u - cfg.pad
            xs, xe = max(0, -ro), min(oh, cfg.H - ro)
            if xs < xe and ys < ye:
                total += (xe - xs) * (ye - ys)
    return cfg.N * cfg.K * cfg.C * total


def direct_forward(d, g, cfg: LayerConfig, accum: Precision = Precision.FP64,
                   counter: Optional[OpCounter] = None) -> Tensor4:
    """Direct correlation with zero padding; output (N, K, out_h, out_w) in the
    accumulator precision (direct.py:82-114).  Same ValueErrors."""
    if accum not in (Precision.FP32, Precision.FP64):
        raise ValueError("accumulator precision must be fp32 or fp64")
    if tuple(d.shape) != (cfg.N, cfg.C, cfg.H, cfg.W):
        raise ValueError(f"data shape {d.shape} does not match {cfg}")
    if tuple(g.shape) != (cfg.K, cfg.C, cfg.R, cfg.S):
        raise ValueError(f"filter shape {g.shape} does not match {cfg}")
    import torch
    dp = precision_of(d)
    in_dt = np.float64 if dp is Precision.FP64 else np.float32
    in_id = _lib.PREC_FP64 if dp is Precision.FP64 else _lib.PREC_FP32
    acc_id = _lib.PREC_FP64 if accum is Precision.FP64 else _lib.PREC_FP32
    d_dev = torch.from_numpy(np.array(d.data, dtype=in_dt, order="C")).cuda()
    g_dev = torch.from_numpy(np.array(g.data, dtype=in_dt, order="C")).cuda()
    y = torch.empty((cfg.N, cfg.K, cfg.out_h, cfg.out_w),
                    dtype=torch.float64 if accum is Precision.FP64 else torch.float32,
                    device="cuda")
    desc = _lib.LayerDesc(cfg.N, cfg.C, cfg.H, cfg.W, cfg.K, cfg.R, cfg.S, cfg.pad)
    _lib.check(_lib.lib.wino_direct_forward(ctypes.byref(desc), in_id, acc_id, d_dev.data_ptr(),
                                            g_dev.data_ptr(), y.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream),
               "wino_direct_forward")
    if counter is not None:
        counter.add("mul", _valid_taps(cfg))
    return Tensor4._wrap(y.cpu().numpy(), accum)
