"""Layer shape descriptor, algorithm descriptors and multiply counter
(mirrors winoconv/direct.py:32-66,179-183, winograd.py:31-236,
counters.py:21-42)."""
from __future__ import annotations

from dataclasses import dataclass, replace
from fractions import Fraction
from typing import Tuple


@dataclass(frozen=True)
class LayerConfig:
    """N images, C in-channels, K filters, H x W, R x S taps, pad, depth (direct.py:32-66)."""

    N: int
    C: int
    H: int
    W: int
    K: int
    R: int = 3
    S: int = 3
    pad: int = 0
    depth: int = 1

    def __post_init__(self) -> None:
        for name in ("N", "C", "H", "W", "K", "R", "S", "depth"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.pad < 0:
            raise ValueError("pad must be >= 0")
        if self.out_h < 1 or self.out_w < 1:
            raise ValueError("output dimensions must be >= 1")

    @property
    def out_h(self) -> int:
        return self.H + 2 * self.pad - self.R + 1

    @property
    def out_w(self) -> int:
        return self.W + 2 * self.pad - self.S + 1

    def with_batch(self, n: int) -> "LayerConfig":
        return replace(self, N=n)


def gflops_direct(cfg: LayerConfig) -> float:
    """Direct-conv GFLOPs, 2 per MAC, depth-weighted (direct.py:179-183)."""
    return 2.0 * cfg.N * cfg.C * cfg.K * cfg.out_h * cfg.out_w * cfg.R * cfg.S / 1e9 * cfg.depth


_F = Fraction
_EXACT = {
    (2, 3): (((1, 0, -1, 0), (0, 1, 1, 0), (0, -1, 1, 0), (0, 1, 0, -1)),
             ((1, 0, 0), (_F(1, 2), _F(1, 2), _F(1, 2)), (_F(1, 2), _F(-1, 2), _F(1, 2)), (0, 0, 1)),
             ((1, 1, 1, 0), (0, 1, -1, -1))),
    # F(3,2): the weight-gradient algorithm F(3x3, 2x2) (winograd.py:171-189)
    (3, 2): (((1, 0, -1, 0), (0, 1, 1, 0), (0, -1, 1, 0), (0, -1, 0, 1)),
             ((1, 0), (_F(1, 2), _F(1, 2)), (_F(1, 2), _F(-1, 2)), (0, 1)),
             ((1, 1, 1, 0), (0, 1, -1, 0), (0, 1, 1, 1))),
    (4, 3): (((4, 0, -5, 0, 1, 0), (0, -4, -4, 1, 1, 0), (0, 4, -4, -1, 1, 0),
              (0, -2, -1, 2, 1, 0), (0, 2, -1, -2, 1, 0), (0, 4, 0, -5, 0, 1)),
             ((_F(1, 4), 0, 0), (_F(-1, 6), _F(-1, 6), _F(-1, 6)), (_F(-1, 6), _F(1, 6), _F(-1, 6)),
              (_F(1, 24), _F(1, 12), _F(1, 6)), (_F(1, 24), _F(-1, 12), _F(1, 6)), (0, 0, 1)),
             ((1, 1, 1, 1, 1, 0), (0, 1, -1, 2, -2, 0), (0, 1, 1, 4, 4, 0), (0, 1, -1, 8, -8, 1))),
}
_FLOPS_1D = {(2, 3): (4, 4, 4), (4, 3): (13, 8, 10)}


@dataclass(frozen=True)
class WinogradAlgorithm:
    """F(m, r) descriptor.  The matrices are the reference's exact rationals
    (winograd.py:151-215); the CUDA kernels compile the same constants in
    (csrc/winograd_mats.cuh)."""

    m: int
    r: int
    BT: Tuple[Tuple[Fraction, ...], ...]
    G: Tuple[Tuple[Fraction, ...], ...]
    AT: Tuple[Tuple[Fraction, ...], ...]
    flops_1d: Tuple[int, int, int] | None = None
    name: str = ""

    @property
    def alpha(self) -> int:
        return self.m + self.r - 1

    @property
    def label(self) -> str:
        return self.name or f"F({self.m},{self.r})"

    def transform_flop_counts(self) -> Tuple[int, int, int]:
        """2D (data, filter, inverse) per-tile costs from 1D (winograd.py:116-131)."""
        b, g, d = self.flops_1d
        return b * 2 * self.alpha, g * (self.r + self.alpha), d * (self.m + self.alpha)

    def lowered(self, dtype) -> tuple:
        import numpy as np
        low = lambda rows: np.array([[float(Fraction(v)) for v in row] for row in rows], dtype=dtype)
        return low(self.BT), low(self.G), low(self.AT)


def builtin(m: int, r: int) -> WinogradAlgorithm:
    """Builtin F(m, r) (winograd.py:225-232): (2,3) and (4,3) for the forward,
    (3,2) for the weight gradient."""
    try:
        bt, g, at = _EXACT[(m, r)]
    except KeyError:
        raise KeyError(f"no builtin algorithm for F({m},{r}); available: "
                       f"{sorted(_EXACT)}") from None
    conv = lambda rows: tuple(tuple(Fraction(v) for v in row) for row in rows)
    return WinogradAlgorithm(m=m, r=r, BT=conv(bt), G=conv(g), AT=conv(at),
                             flops_1d=_FLOPS_1D.get((m, r)), name=f"F({m},{r})")


def builtin_sizes():
    return tuple(sorted(_EXACT))


class OpCounter:
    """Additive operation tally (counters.py:21-42)."""

    __slots__ = ("counts",)

    def __init__(self) -> None:
        self.counts: dict = {}

    def add(self, key: str, n: int = 1) -> None:
        if n < 0:
            raise ValueError("counter increments must be non-negative")
        self.counts[key] = self.counts.get(key, 0) + n

    def get(self, key: str) -> int:
        return self.counts.get(key, 0)

    def __getitem__(self, key: str) -> int:
        return self.get(key)

    def __repr__(self) -> str:
        return "OpCounter(" + ", ".join(f"{k}={v}" for k, v in sorted(self.counts.items())) + ")"
