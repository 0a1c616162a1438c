"""ctypes binding of libwino.so (include/wino.h).

The CUDA library is the product: there is no CPU fallback.  If the shared
object is missing the import of this module fails loudly; if no GPU is
present, calls into it fail with RuntimeError from the CUDA status.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwino.so")

WINO_OK, WINO_EINVAL, WINO_EUNSUPPORTED, WINO_ENOMEM, WINO_ECUDA = 0, 1, 2, 3, 4

PREC_FP32, PREC_TF32, PREC_BF16, PREC_FP16, PREC_FP64 = 0, 1, 2, 3, 4
PREC_BY_NAME = {"fp32": PREC_FP32, "3xtf32": PREC_FP32, "tf32": PREC_TF32,
                "bf16": PREC_BF16, "fp16": PREC_FP16, "fp64": PREC_FP64}
PREC_NAME = {PREC_FP32: "fp32", PREC_TF32: "tf32", PREC_BF16: "bf16",
             PREC_FP16: "fp16", PREC_FP64: "fp64"}

# Every symbol include/wino.h declares (checked by tests/test_abi.py).
EXPORTED = ("wino_plan_create", "wino_plan_destroy", "wino_plan_get_info",
            "wino_filter_transform", "wino_forward", "wino_forward_host", "wino_forward_timed",
            "wino_timer_create", "wino_timer_destroy", "wino_timer_break", "wino_timer_read",
            "wino_wgrad_workspace", "wino_grad_weights", "wino_direct_forward", "wino_relu_pool",
            "wino_fft_workspace", "wino_fft_forward", "wino_forward_act",
            "wino_shard_bounds", "wino_shard_workspace", "wino_forward_sharded",
            "wino_last_error", "wino_version")


class LayerDesc(ctypes.Structure):
    """wino_layer_t"""
    _fields_ = [(n, ctypes.c_int) for n in ("N", "C", "H", "W", "K", "R", "S", "pad")]


class PlanInfo(ctypes.Structure):
    """wino_plan_info_t"""
    _fields_ = [
        ("m", ctypes.c_int), ("r", ctypes.c_int), ("alpha", ctypes.c_int),
        ("out_h", ctypes.c_int), ("out_w", ctypes.c_int),
        ("tiles_h", ctypes.c_int), ("tiles_w", ctypes.c_int),
        ("P", ctypes.c_longlong),
        ("prec", ctypes.c_int), ("c_pad", ctypes.c_int), ("op_bytes", ctypes.c_int),
        ("op_splits", ctypes.c_int),
        ("gemm_bn", ctypes.c_int), ("gemm_splits", ctypes.c_int),
        ("rows_per_chunk", ctypes.c_int), ("num_chunks", ctypes.c_int),
        ("chunk_tiles", ctypes.c_longlong),
        ("u_bytes", ctypes.c_size_t), ("workspace_bytes", ctypes.c_size_t),
        ("launches_per_forward", ctypes.c_int), ("fused_small_c", ctypes.c_int),
        ("multiplies", ctypes.c_longlong),
        ("fused", ctypes.c_int), ("fused_splits", ctypes.c_int),
        ("m_bytes_per_elem", ctypes.c_int), ("combined_transforms", ctypes.c_int),
        ("staging_bytes", ctypes.c_size_t),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA extension has not been built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`). "
            "There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    vp, c_int, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    lib.wino_plan_create.argtypes = [ctypes.POINTER(LayerDesc), c_int, c_int, sz,
                                     ctypes.POINTER(vp)]
    lib.wino_plan_destroy.argtypes = [vp]
    lib.wino_plan_get_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
    lib.wino_filter_transform.argtypes = [vp, vp, vp, vp]
    lib.wino_forward.argtypes = [vp, vp, vp, vp, vp, vp, sz, vp]
    lib.wino_forward_host.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.wino_forward_timed.argtypes = [vp, vp, vp, vp, vp, vp, sz, vp, vp]
    lib.wino_timer_create.argtypes = [ctypes.POINTER(vp)]
    lib.wino_timer_destroy.argtypes = [vp]
    lib.wino_timer_break.argtypes = [vp]
    lib.wino_timer_read.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(c_int)]
    lib.wino_wgrad_workspace.argtypes = [ctypes.POINTER(LayerDesc), c_int, sz,
                                         ctypes.POINTER(sz)]
    lib.wino_grad_weights.argtypes = [ctypes.POINTER(LayerDesc), c_int, vp, vp, vp, vp, sz, sz,
                                      vp]
    lib.wino_direct_forward.argtypes = [ctypes.POINTER(LayerDesc), c_int, c_int, vp, vp, vp, vp]
    lib.wino_fft_workspace.argtypes = [ctypes.POINTER(LayerDesc), c_int, ctypes.POINTER(sz)]
    lib.wino_fft_forward.argtypes = [ctypes.POINTER(LayerDesc), c_int, c_int, vp, vp, vp, vp, sz,
                                     vp]
    lib.wino_relu_pool.argtypes = [vp, vp, c_int, c_int, c_int, c_int, c_int, vp]
    lib.wino_forward_act.argtypes = [vp, vp, vp, vp, vp, vp, sz, c_int, vp]
    pint = ctypes.POINTER(c_int)
    lib.wino_shard_bounds.argtypes = [c_int, c_int, c_int, pint, pint]
    lib.wino_shard_workspace.argtypes = [vp, c_int, c_int, c_int, ctypes.POINTER(sz)]
    lib.wino_forward_sharded.argtypes = [vp, c_int, pint] + [ctypes.POINTER(vp)] * 5 + [
        ctypes.POINTER(sz), ctypes.POINTER(vp)]
    lib.wino_last_error.restype = ctypes.c_char_p
    lib.wino_version.restype = ctypes.c_char_p
    for name in EXPORTED:
        if name not in ("wino_last_error", "wino_version"):
            getattr(lib, name).restype = c_int
    return lib


lib = _load()


def check(rc: int, what: str = "") -> None:
    """Map a wino status code onto the reference's exception types."""
    if rc == WINO_OK:
        return
    msg = lib.wino_last_error().decode(errors="replace") or what
    if rc in (WINO_EINVAL, WINO_EUNSUPPORTED):
        raise ValueError(msg)
    if rc == WINO_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


def version() -> str:
    return lib.wino_version().decode()
