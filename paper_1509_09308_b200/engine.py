"""Whole-layer Winograd convolution on B200 -- the drop-in for
``winoconv.engine`` (/root/reference/pkg/src/winoconv/engine.py).

Two levels:

* ``WinogradPlan`` -- device-level object over the C ABI (``include/wino.h``):
  device tensors in, device tensors out, explicit stream, reusable workspace.
  This is what the bench, the multi-GPU driver and CUDA-graph capture use.
* ``winograd_forward(d, g, cfg, alg, cache_filters, counter, cache)`` -- the
  reference's signature and semantics (engine.py:198-254) on host ``Tensor4``
  data: validation errors, FX filter cache, multiply counter, fresh read-only
  output.  It runs the CUDA path; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import threading
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from . import _lib
from .layer import LayerConfig, OpCounter, WinogradAlgorithm, builtin
from .tensors import Precision, Tensor4, precision_of

# --------------------------------------------------------------------- tiles


@dataclass(frozen=True)
class TileGrid:
    """Row-major tile enumeration (engine.py:40-80): tile b <-> (n, ty, tx);
    its alpha x alpha input patch starts at (m*ty - pad, m*tx - pad)."""

    m: int
    r: int
    N: int
    tiles_h: int
    tiles_w: int
    pad: int

    @classmethod
    def for_layer(cls, cfg: LayerConfig, m: int, r: int) -> "TileGrid":
        return cls(m=m, r=r, N=cfg.N, tiles_h=-(-cfg.out_h // m), tiles_w=-(-cfg.out_w // m),
                   pad=cfg.pad)

    @property
    def alpha(self) -> int:
        return self.m + self.r - 1

    @property
    def P(self) -> int:
        return self.N * self.tiles_h * self.tiles_w

    def index(self, b: int) -> Tuple[int, int, int]:
        if not 0 <= b < self.P:
            raise IndexError(f"tile {b} out of range [0, {self.P})")
        n, rest = divmod(b, self.tiles_h * self.tiles_w)
        ty, tx = divmod(rest, self.tiles_w)
        return n, ty, tx

    def origin(self, b: int) -> Tuple[int, int]:
        _, ty, tx = self.index(b)
        return self.m * ty - self.pad, self.m * tx - self.pad


def tile_count(cfg: LayerConfig, m: int) -> int:
    """P = N * ceil(outH/m) * ceil(outW/m) (engine.py:83-87)."""
    if m < 1:
        raise ValueError(f"need m >= 1, got {m}")
    return cfg.N * (-(-cfg.out_h // m)) * (-(-cfg.out_w // m))


def multiply_stage_flops(cfg: LayerConfig, m: int) -> int:
    """P*C*K*(m+R-1)*(m+S-1) real multiplies in the GEMM stage (engine.py:90-95)."""
    return tile_count(cfg, m) * cfg.C * cfg.K * (m + cfg.R - 1) * (m + cfg.S - 1)


# --------------------------------------------------------------------- plan

def _torch():
    import torch
    return torch


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        return _torch().cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


class WinogradPlan:
    """One layer shape x algorithm x precision, over ``wino_plan_t``.

    Plan creation (and ``info``) is host-only and works without a GPU;
    everything that launches kernels needs ``cuda`` device tensors.
    """

    def __init__(self, cfg: LayerConfig, m: int, prec: str = "fp32",
                 workspace_limit: int = 0) -> None:
        if prec not in _lib.PREC_BY_NAME:
            raise ValueError(f"unknown precision {prec!r}; known: {sorted(_lib.PREC_BY_NAME)}")
        self.cfg = cfg
        self.m = m
        self.prec = _lib.PREC_NAME[_lib.PREC_BY_NAME[prec]]
        self._prec_id = _lib.PREC_BY_NAME[prec]
        desc = _lib.LayerDesc(cfg.N, cfg.C, cfg.H, cfg.W, cfg.K, cfg.R, cfg.S, cfg.pad)
        handle = ctypes.c_void_p()
        _lib.check(_lib.lib.wino_plan_create(ctypes.byref(desc), m, self._prec_id,
                                             int(workspace_limit), ctypes.byref(handle)),
                   "wino_plan_create")
        self._h = handle
        info = _lib.PlanInfo()
        _lib.check(_lib.lib.wino_plan_get_info(self._h, ctypes.byref(info)))
        self.info = info.as_dict()

    def __del__(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and _lib.lib is not None:
            _lib.lib.wino_plan_destroy(h)
            self._h = None

    # dtype of data/outputs
    @property
    def data_dtype(self):
        return _torch().float64 if self._prec_id == _lib.PREC_FP64 else _torch().float32

    @property
    def out_shape(self) -> Tuple[int, int, int, int]:
        c = self.cfg
        return (c.N, c.K, c.out_h, c.out_w)

    @property
    def workspace_bytes(self) -> int:
        return int(self.info["workspace_bytes"])

    @property
    def u_bytes(self) -> int:
        return int(self.info["u_bytes"])

    def alloc_workspace(self, device=None):
        t = _torch()
        return t.empty(self.workspace_bytes, dtype=t.uint8, device=device or "cuda")

    def _check_dev(self, x, shape, name):
        t = _torch()
        if not isinstance(x, t.Tensor) or not x.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if tuple(x.shape) != tuple(shape) or x.dtype != self.data_dtype or not x.is_contiguous():
            raise ValueError(f"{name}: expected contiguous {self.data_dtype} {tuple(shape)}, got "
                             f"{x.dtype} {tuple(x.shape)}")

    def filter_transform(self, g, U=None, stream=None):
        """G g G^T into the operand-format U stack (engine.py:104-114)."""
        t = _torch()
        c = self.cfg
        self._check_dev(g, (c.K, c.C, c.R, c.S), "g")
        if U is None:
            U = t.empty(self.u_bytes, dtype=t.uint8, device=g.device)
        _lib.check(_lib.lib.wino_filter_transform(self._h, g.data_ptr(), U.data_ptr(),
                                                  _stream_handle(stream)), "filter transform")
        return U

    def _check_host(self, x, shape, name):
        t = _torch()
        if not isinstance(x, t.Tensor) or x.is_cuda:
            raise ValueError(f"{name} must be a host (CPU) tensor")
        if tuple(x.shape) != tuple(shape) or x.dtype != self.data_dtype or not x.is_contiguous():
            raise ValueError(f"{name}: expected contiguous {self.data_dtype} {tuple(shape)}, got "
                             f"{x.dtype} {tuple(x.shape)}")
        if not x.is_pinned():
            raise ValueError(f"{name} must be in pinned host memory (asynchronous copies)")

    def _operands(self, d, y, U, g, workspace, stream, out_shape=None):
        """Validate the device operands of one forward; allocate y / workspace when
        absent.  Fresh allocations are made on torch's current stream, so when
        the launch stream differs they are recorded on it (the caching allocator
        then keeps them alive until the launch stream's work is done)."""
        t = _torch()
        c = self.cfg
        self._check_dev(d, (c.N, c.C, c.H, c.W), "d")
        if U is None and g is None:
            raise ValueError("need U or g")
        if U is not None:
            if not isinstance(U, t.Tensor) or not U.is_cuda or not U.is_contiguous():
                raise ValueError("U must be a contiguous CUDA tensor")
            if U.numel() * U.element_size() < self.u_bytes:
                raise ValueError(f"U: {U.numel() * U.element_size()} bytes, plan needs "
                                 f"{self.u_bytes}")
        else:
            self._check_dev(g, (c.K, c.C, c.R, c.S), "g")
        fresh = []
        out_shape = self.out_shape if out_shape is None else out_shape
        if y is None:
            y = t.empty(out_shape, dtype=self.data_dtype, device=d.device)
            fresh.append(y)
        else:
            self._check_dev(y, out_shape, "y")
        if workspace is None:
            workspace = self.alloc_workspace(d.device)
            fresh.append(workspace)
        else:
            if (not isinstance(workspace, t.Tensor) or not workspace.is_cuda
                    or not workspace.is_contiguous()):
                raise ValueError("workspace must be a contiguous CUDA tensor")
            if workspace.numel() * workspace.element_size() < self.workspace_bytes:
                raise ValueError(f"workspace: {workspace.numel() * workspace.element_size()} "
                                 f"bytes, plan needs {self.workspace_bytes}")
        if stream is not None and fresh:
            ts = stream if isinstance(stream, t.cuda.Stream) else None
            if ts is not None and ts != t.cuda.current_stream(d.device):
                for x in fresh:
                    x.record_stream(ts)
        return y, workspace

    @staticmethod
    def _ptr(x):
        return x.data_ptr() if x is not None else None

    ACTS = {None: 0, "relu": 1, "relu_pool": 2}

    def act_shape(self, act=None):
        """Output shape of forward(act=...): relu_pool halves out_h and out_w."""
        N, K, oh, ow = self.out_shape
        return (N, K, oh // 2, ow // 2) if act == "relu_pool" else (N, K, oh, ow)

    def forward(self, d, y=None, U=None, g=None, workspace=None, stream=None, act=None):
        """y = conv(d, g) with the precomputed U (FX) or transforming g in place.
        act="relu" / "relu_pool" fuses max(y, 0) / relu + 2x2 max-pool into the
        output transform's stores (wino_forward_act)."""
        if act not in self.ACTS:
            raise ValueError(f"act must be one of {list(self.ACTS)}, got {act!r}")
        y, workspace = self._operands(d, y, U, g, workspace, stream, self.act_shape(act))
        args = (self._h, d.data_ptr(), self._ptr(U), g.data_ptr() if U is None else None,
                y.data_ptr(), workspace.data_ptr(), workspace.numel() * workspace.element_size())
        if act is None:
            _lib.check(_lib.lib.wino_forward(*args, _stream_handle(stream)), "wino_forward")
        else:
            _lib.check(_lib.lib.wino_forward_act(*args, self.ACTS[act], _stream_handle(stream)),
                       "wino_forward_act")
        return y

    def forward_timed(self, d, y, timer: "StageTimer", U=None, g=None, workspace=None,
                      stream=None):
        """forward() plus one CUDA event per launch into `timer` (asynchronous)."""
        y, workspace = self._operands(d, y, U, g, workspace, stream)
        _lib.check(_lib.lib.wino_forward_timed(
            self._h, d.data_ptr(), self._ptr(U), g.data_ptr() if U is None else None,
            y.data_ptr(), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
            _stream_handle(stream), timer._h), "wino_forward_timed")
        return y

    def forward_host(self, d_host, y_host, d_dev, y_dev, U=None, g=None, workspace=None,
                     stream=None):
        """End-to-end call with host buffers (pinned, for asynchronous copies):
        H2D of d_host into d_dev, the forward, D2H of y_dev into y_host."""
        c = self.cfg
        self._check_host(d_host, (c.N, c.C, c.H, c.W), "d_host")
        self._check_host(y_host, self.out_shape, "y_host")
        y_dev, workspace = self._operands(d_dev, y_dev, U, g, workspace, stream)
        _lib.check(_lib.lib.wino_forward_host(
            self._h, d_host.data_ptr(), self._ptr(U), g.data_ptr() if U is None else None,
            y_host.data_ptr(), d_dev.data_ptr(), y_dev.data_ptr(), workspace.data_ptr(),
            workspace.numel() * workspace.element_size(), _stream_handle(stream)),
            "wino_forward_host")
        return y_host


class StageTimer:
    """Device-side per-stage timing of forwards (wino_timer_t)."""

    STAGES = ("filter_transform", "input_transform", "batched_gemm", "output_transform")

    def __init__(self) -> None:
        h = ctypes.c_void_p()
        _lib.check(_lib.lib.wino_timer_create(ctypes.byref(h)), "wino_timer_create")
        self._h = h

    def gap(self) -> None:
        _lib.check(_lib.lib.wino_timer_break(self._h))

    def read(self):
        """Synchronise; returns (stage_ms[4], launches[4]) accumulated since last read."""
        ms = (ctypes.c_float * 4)()
        n = (ctypes.c_int * 4)()
        _lib.check(_lib.lib.wino_timer_read(self._h, ms, n), "wino_timer_read")
        return list(ms), list(n)

    def __del__(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and _lib.lib is not None:
            _lib.lib.wino_timer_destroy(h)
            self._h = None


_plans: dict = {}
_plans_lock = threading.Lock()


def get_plan(cfg: LayerConfig, m: int, prec: str, workspace_limit: int = 0) -> WinogradPlan:
    # WINO_PATH (staged / fused / hybrid) is read by the C planner at plan creation
    key = (cfg.N, cfg.C, cfg.H, cfg.W, cfg.K, cfg.R, cfg.S, cfg.pad, m, prec, workspace_limit,
           os.environ.get("WINO_PATH", ""))
    with _plans_lock:
        plan = _plans.get(key)
        if plan is None:
            plan = WinogradPlan(cfg, m, prec, workspace_limit)
            _plans[key] = plan
        return plan


def default_prec(precision: Precision) -> str:
    """Reference semantics: arithmetic in the data type (engine.py:220-254).
    fp32 / fp16-sim data -> fp32-accurate 3xTF32 tensor-core GEMM; fp64 -> fp64."""
    return "fp64" if precision is Precision.FP64 else "fp32"


# --------------------------------------------------------------------- FX cache

class FilterCache:
    """Keyed store of device-resident transformed filter stacks (engine.py:117-160).

    Key = (sha1 of the lowered G, dtype, shape, sha1 of the filter bytes, operand
    precision): a hit returns the bit-identical U a fresh transform would give.
    """

    def __init__(self) -> None:
        self._store: dict = {}
        self._scalars: dict = {}
        self.hits = 0
        self.misses = 0
        self._lock = threading.Lock()

    @staticmethod
    def _key(g: Tensor4, alg: WinogradAlgorithm, prec: str) -> tuple:
        dt = g.data.dtype
        alg_tag = hashlib.sha1(alg.lowered(dt)[1].tobytes()).hexdigest()
        g_tag = hashlib.sha1(np.ascontiguousarray(g.data).tobytes()).hexdigest()
        return (alg_tag, np.dtype(dt).str, tuple(g.shape), g_tag, prec)

    def fetch(self, g: Tensor4, alg: WinogradAlgorithm, counter: Optional[OpCounter] = None,
              prec: Optional[str] = None, plan: Optional[WinogradPlan] = None):
        prec = prec or default_prec(precision_of(g))
        key = self._key(g, alg, prec)
        with self._lock:
            hit = self._store.get(key)
            if hit is not None:
                self.hits += 1
                return hit
            self.misses += 1
        K, C, R, S = g.shape
        if plan is None:
            # U depends only on (K, C, m, prec): any layer with these filters works
            plan = get_plan(LayerConfig(N=1, C=C, H=R, W=S, K=K, R=R, S=S, pad=1), alg.m, prec)
        t = _torch()
        g_dev = t.from_numpy(np.array(g.data, order="C")).to("cuda")
        U = plan.filter_transform(g_dev)
        with self._lock:
            self._store[key] = U
            self._scalars[key] = alg.alpha * alg.alpha * K * C
        return U

    def workspace_scalars(self) -> int:
        """Cached footprint: alpha^2*K*C scalars per entry (engine.py:150-152)."""
        return sum(self._scalars.values())

    def clear(self) -> None:
        with self._lock:
            self._store.clear()
            self._scalars.clear()
            self.hits = 0
            self.misses = 0

    def __len__(self) -> int:
        return len(self._store)


_shared_cache = FilterCache()


def shared_filter_cache() -> FilterCache:
    return _shared_cache


# --------------------------------------------------------------------- forward

def _out_precision(precision: Precision) -> Precision:
    return Precision.FP64 if precision is Precision.FP64 else Precision.FP32


def winograd_forward(d, g, cfg: LayerConfig, alg: Optional[WinogradAlgorithm] = None,
                     cache_filters: bool = False, counter: Optional[OpCounter] = None,
                     cache: Optional[FilterCache] = None, prec: Optional[str] = None) -> Tensor4:
    """F(m x m, 3 x 3) layer forward on the GPU (engine.py:198-254).

    ``prec`` (extension) picks the transform-space GEMM arithmetic: ``"fp32"``
    (3xTF32, default for fp32 data), ``"tf32"``, ``"bf16"``, ``"fp16"``, or
    ``"fp64"`` (default for fp64 data).
    """
    if alg is None:
        alg = builtin(2, 3)
    dp, gp = precision_of(d), precision_of(g)
    if dp != gp:
        raise ValueError(f"mixed precisions: {dp} vs {gp}")
    if tuple(d.shape) != (cfg.N, cfg.C, cfg.H, cfg.W):
        raise ValueError(f"data shape {d.shape} does not match {cfg}")
    if tuple(g.shape) != (cfg.K, cfg.C, cfg.R, cfg.S):
        raise ValueError(f"filter shape {g.shape} does not match {cfg}")
    if cfg.R != alg.r or cfg.S != alg.r:
        raise ValueError(f"layer filter {cfg.R}x{cfg.S} but algorithm is F({alg.m},{alg.r})")
    if (alg.m, alg.r) not in ((2, 3), (4, 3)):
        raise ValueError(f"GPU path implements F(2,3) and F(4,3), not {alg.label}")
    prec = prec or default_prec(dp)
    if (prec == "fp64") != (dp is Precision.FP64):
        raise ValueError(f"prec {prec!r} does not match data precision {dp.value}")
    t = _torch()
    plan = get_plan(cfg, alg.m, prec)
    d_dev = t.from_numpy(np.array(d.data, order="C")).to("cuda")
    if cache_filters:
        store = cache if cache is not None else _shared_cache
        U = store.fetch(g, alg, counter=counter, prec=prec, plan=plan)
        y = plan.forward(d_dev, U=U)
    else:
        g_dev = t.from_numpy(np.array(g.data, order="C")).to("cuda")
        y = plan.forward(d_dev, g=g_dev)
    if counter is not None:  # kernels.py:63-64 semantics
        counter.add("mul", multiply_stage_flops(cfg, alg.m))
    out = y.cpu().numpy()
    return Tensor4._wrap(out, _out_precision(dp))


def winograd_grad_inputs(dy, g, cfg: LayerConfig, alg: Optional[WinogradAlgorithm] = None,
                         cache_filters: bool = False, counter: Optional[OpCounter] = None,
                         cache: Optional[FilterCache] = None, prec: Optional[str] = None) -> Tensor4:
    """dL/dInput = the forward over dY with flipped, (k,c)-swapped filters and
    pad' = R-1-pad (engine.py:257-275) -- the same CUDA path."""
    if cfg.pad > cfg.R - 1:
        raise ValueError(f"pad={cfg.pad} exceeds R-1={cfg.R - 1}; gradient tiling undefined")
    if tuple(dy.shape) != (cfg.N, cfg.K, cfg.out_h, cfg.out_w):
        raise ValueError(f"dY shape {dy.shape} does not match {cfg}")
    flipped = np.ascontiguousarray(g.data[:, :, ::-1, ::-1].transpose(1, 0, 2, 3))
    gt = Tensor4._wrap(flipped, precision_of(g))
    adj = LayerConfig(N=cfg.N, C=cfg.K, H=cfg.out_h, W=cfg.out_w, K=cfg.C, R=cfg.R, S=cfg.S,
                      pad=cfg.R - 1 - cfg.pad)
    dd = winograd_forward(dy, gt, adj, alg=alg, cache_filters=cache_filters, counter=counter,
                          cache=cache, prec=prec)
    if tuple(dd.shape) != (cfg.N, cfg.C, cfg.H, cfg.W):
        raise AssertionError(f"input gradient came out {dd.shape}")
    return dd


# --------------------------------------------------------------------- dL/dg

def grad_weights_device(d, dy, cfg: LayerConfig, prec: str = "fp32", workspace=None,
                        workspace_limit: int = 0, stream=None):
    """Device-level weight gradient (C ABI ``wino_grad_weights``): d (N,C,H,W)
    and dy (N,K,out_h,out_w) CUDA tensors -> dg (K,C,3,3) CUDA tensor."""
    t = _torch()
    if prec not in _lib.PREC_BY_NAME:
        raise ValueError(f"unknown precision {prec!r}")
    pid = _lib.PREC_BY_NAME[prec]
    dt = t.float64 if pid == _lib.PREC_FP64 else t.float32
    for x, shape, name in ((d, (cfg.N, cfg.C, cfg.H, cfg.W), "d"),
                           (dy, (cfg.N, cfg.K, cfg.out_h, cfg.out_w), "dy")):
        if not isinstance(x, t.Tensor) or not x.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if tuple(x.shape) != shape or x.dtype != dt or not x.is_contiguous():
            raise ValueError(f"{name}: expected contiguous {dt} {shape}, got {x.dtype} "
                             f"{tuple(x.shape)}")
    desc = _lib.LayerDesc(cfg.N, cfg.C, cfg.H, cfg.W, cfg.K, cfg.R, cfg.S, cfg.pad)
    need = ctypes.c_size_t()
    _lib.check(_lib.lib.wino_wgrad_workspace(ctypes.byref(desc), pid, int(workspace_limit),
                                             ctypes.byref(need)), "wino_wgrad_workspace")
    if workspace is None or workspace.numel() < need.value:
        workspace = t.empty(need.value, dtype=t.uint8, device=d.device)
    dg = t.empty((cfg.K, cfg.C, cfg.R, cfg.S), dtype=dt, device=d.device)
    _lib.check(_lib.lib.wino_grad_weights(ctypes.byref(desc), pid, d.data_ptr(), dy.data_ptr(),
                                          dg.data_ptr(), workspace.data_ptr(),
                                          workspace.numel(), int(workspace_limit),
                                          _stream_handle(stream)), "wino_grad_weights")
    return dg


def winograd_grad_weights(d, dy, cfg: LayerConfig, alg_w: Optional[WinogradAlgorithm] = None,
                          counter: Optional[OpCounter] = None, prec: Optional[str] = None) -> Tensor4:
    """dL/dFilter via F(3x3, 2x2) on the GPU (engine.py:278-328): same
    validation and exceptions, counter ``"mul" += 16*K*B*C`` (the reference's
    batched_matmul over the tile axis), fresh read-only output."""
    if alg_w is None:
        if cfg.R != 3 or cfg.S != 3:
            raise ValueError(f"default weight-gradient algorithm needs R=S=3, "
                             f"got {cfg.R}x{cfg.S}")
        alg_w = builtin(3, 2)
    if alg_w.m != cfg.R or cfg.R != cfg.S:
        raise ValueError(f"algorithm F({alg_w.m},{alg_w.r}) cannot produce "
                         f"{cfg.R}x{cfg.S} gradients")
    if (alg_w.m, alg_w.r) != (3, 2):
        raise ValueError(f"GPU path implements F(3,2) for weight gradients, not {alg_w.label}")
    dp, yp = precision_of(d), precision_of(dy)
    if dp != yp:
        raise ValueError(f"mixed precisions: {dp} vs {yp}")
    if tuple(d.shape) != (cfg.N, cfg.C, cfg.H, cfg.W):
        raise ValueError(f"data shape {d.shape} does not match {cfg}")
    if tuple(dy.shape) != (cfg.N, cfg.K, cfg.out_h, cfg.out_w):
        raise ValueError(f"dY shape {dy.shape} does not match {cfg}")
    prec = prec or default_prec(dp)
    if (prec == "fp64") != (dp is Precision.FP64):
        raise ValueError(f"prec {prec!r} does not match data precision {dp.value}")
    t = _torch()
    d_dev = t.from_numpy(np.array(d.data, order="C")).to("cuda")
    y_dev = t.from_numpy(np.array(dy.data, order="C")).to("cuda")
    dg = grad_weights_device(d_dev, y_dev, cfg, prec)
    if counter is not None:
        B = cfg.N * (-(-cfg.out_h // 2)) * (-(-cfg.out_w // 2))
        counter.add("mul", 16 * cfg.K * B * cfg.C)
    return Tensor4._wrap(dg.cpu().numpy(), _out_precision(dp))
