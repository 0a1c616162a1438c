"""Algorithm-name dispatch, the accuracy harness and the layer benchmark on the
GPU path (mirrors winoconv/commands.py:25-178).

Algorithm names are the reference's (``direct``, ``direct-fp32``, ``f2x2``,
``f4x4``, ``f2x2-fx``, ``f4x4-fx``, ``fft``); the Winograd names take an
optional GEMM precision suffix, e.g. ``f4x4-fx:bf16``.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

from .direct import direct_forward
from .engine import FilterCache, get_plan, winograd_forward
from .fftconv import fft_forward_layer
from .layer import LayerConfig, builtin, gflops_direct
from .suites import get_suite
from .tensors import Precision, Tensor4, fill_uniform, max_abs_error, quantize_fp16

WINOGRAD_ALGOS = ("f2x2", "f4x4", "f2x2-fx", "f4x4-fx")
DIRECT_ALGOS = ("direct", "direct-fp32")
BENCH_ALGOS = ("direct", "direct-fp32", "f2x2", "f4x4", "f2x2-fx", "f4x4-fx",
               "fft")  # commands.py:26
ACCURACY_ALGOS = ("direct-fp32", "f2x2", "f4x4", "fft")  # commands.py:25
PRECISIONS = ("fp32", "tf32", "bf16", "fp16", "fp64")


def parse_algo(algo: str) -> Tuple[int, bool, Optional[str]]:
    """'f4x4-fx:bf16' -> (m=4, fx=True, prec='bf16')."""
    base, _, prec = algo.partition(":")
    if base not in WINOGRAD_ALGOS:
        raise ValueError(f"unknown algorithm {algo!r}; known: {', '.join(WINOGRAD_ALGOS)}"
                         " (optionally ':<prec>')")
    if prec and prec not in PRECISIONS:
        raise ValueError(f"unknown precision {prec!r}; known: {', '.join(PRECISIONS)}")
    return (2 if base.startswith("f2x2") else 4), base.endswith("-fx"), (prec or None)


def run_layer(algo: str, d: Tensor4, g: Tensor4, cfg: LayerConfig,
              cache: Optional[FilterCache] = None, counter=None) -> Tensor4:
    """Dispatch one forward layer by algorithm name (commands.py:31-51)."""
    if algo == "direct":
        accum = Precision.FP64 if d.precision is Precision.FP64 else Precision.FP32
        return direct_forward(d, g, cfg, accum=accum, counter=counter)
    if algo == "direct-fp32":
        return direct_forward(d, g, cfg, accum=Precision.FP32, counter=counter)
    if algo == "fft":
        return fft_forward_layer(d, g, cfg, tile=8, counter=counter)
    m, fx, prec = parse_algo(algo)
    return winograd_forward(d, g, cfg, builtin(m, 3), cache_filters=fx, cache=cache,
                            counter=counter, prec=prec)


def layer_inputs(cfg: LayerConfig, seed: int, index: int) -> Tuple[Tensor4, Tensor4]:
    """Data seed seed+2i, filters seed+2i+1, U[-1,1) (commands.py:54-61)."""
    d = fill_uniform(Tensor4.zeros((cfg.N, cfg.C, cfg.H, cfg.W)), seed + 2 * index, -1.0, 1.0)
    g = fill_uniform(Tensor4.zeros((cfg.K, cfg.C, cfg.R, cfg.S)), seed + 2 * index + 1, -1.0, 1.0)
    return d, g


_layer_inputs = layer_inputs


def _parse_cell(c: str):
    if c == "":
        return None
    for conv in (int, float):
        try:
            return conv(c)
        except ValueError:
            pass
    return c


@dataclass
class Report:
    columns: Tuple[str, ...]
    rows: List[tuple] = field(default_factory=list)
    seed: Optional[int] = None

    def add(self, *vals) -> None:
        if len(vals) != len(self.columns):
            raise ValueError("row width mismatch")
        self.rows.append(tuple(vals))

    def to_csv(self) -> str:
        lines = [] if self.seed is None else [f"# seed={self.seed}"]
        lines.append(",".join(self.columns))
        for r in self.rows:
            lines.append(",".join("" if v is None else repr(v) if isinstance(v, float) else str(v)
                                  for v in r))
        return "\n".join(lines) + "\n"

    @classmethod
    def from_csv(cls, text: str) -> "Report":
        """Inverse of to_csv (reports.py:65-85): '# seed=' header, empty cells
        are None, ints and floats (repr round-trips exactly) are parsed back."""
        import csv

        seed = None
        lines = []
        for line in text.splitlines():
            if line.startswith("#"):
                body = line.lstrip("#").strip()
                if body.startswith("seed="):
                    seed = int(body[len("seed="):])
                continue
            if line.strip():
                lines.append(line)
        if not lines:
            raise ValueError("empty report text")
        parsed = list(csv.reader(lines))
        rep = cls(columns=tuple(parsed[0]), seed=seed)
        for raw in parsed[1:]:
            if len(raw) != len(rep.columns):
                raise ValueError(f"row {raw!r} does not match header {rep.columns}")
            rep.rows.append(tuple(_parse_cell(c) for c in raw))
        return rep

    def to_text(self) -> str:
        def fmt(v):
            if v is None:
                return "-"
            return f"{v:.4g}" if isinstance(v, float) else str(v)
        cells = [list(self.columns)] + [[fmt(v) for v in r] for r in self.rows]
        widths = [max(len(row[i]) for row in cells) for i in range(len(self.columns))]
        out = [] if self.seed is None else [f"# seed={self.seed}"]
        for row in cells:
            out.append("  ".join(c.rjust(w) for c, w in zip(row, widths)))
        return "\n".join(out) + "\n"


def _bench_other(algo: str, cfg: LayerConfig, d: Tensor4, g: Tensor4, repeats: int) -> float:
    """Best-of-N seconds of the non-Winograd algorithms (direct, direct-fp32, fft)
    through run_layer -- host Tensor4 in and out, like the reference's timing of
    them (commands.py:160-166): wall clock around a synchronised call."""
    import time

    import torch
    run_layer(algo, d, g, cfg)  # warm-up, untimed
    best = float("inf")
    for _ in range(repeats):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run_layer(algo, d, g, cfg)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def cmd_bench(suite: str = "vgg-e", algo: str = "f2x2", batch: int = 1, repeats: int = 3,
              scale: float = 1.0, seed: int = 0) -> Report:
    """Per-layer best-of-N time and effective GFLOPS = direct-conv GFLOP / time;
    depth-weighted TOTAL row (commands.py:136-178).  Every reference algorithm
    name is accepted (BENCH_ALGOS, commands.py:26).  The Winograd names are
    device-timed (CUDA events, inputs resident in HBM, non-FX names include
    the filter transform); direct / direct-fp32 / fft are timed through
    run_layer around a synchronised call.  Layers that exhaust memory are skipped
    with empty cells."""
    import torch

    if repeats < 1:
        raise ValueError(f"repeats must be >= 1, got {repeats}")
    if algo not in BENCH_ALGOS and algo.partition(":")[0] not in WINOGRAD_ALGOS:
        raise ValueError(f"unknown algorithm {algo!r}; known: {', '.join(BENCH_ALGOS)}")
    wino = algo.partition(":")[0] in WINOGRAD_ALGOS
    if wino:
        m, fx, prec = parse_algo(algo)
    layers = get_suite(suite).scaled(scale).with_batch(batch)
    rep = Report(columns=("layer", "algo", "batch", "msec", "effective_gflops"), seed=seed)
    total_sec = total_gf = 0.0
    for i, entry in enumerate(layers.entries):
        cfg = entry.cfg
        try:
            d, g = layer_inputs(cfg, seed, i)
            if not wino:
                best = _bench_other(algo, cfg, d, g, repeats)
            else:
                plan = get_plan(cfg, m, prec or "fp32")
                d_dev = torch.from_numpy(d.data.copy()).cuda()
                g_dev = torch.from_numpy(g.data.copy()).cuda()
                ws = plan.alloc_workspace()
                y = torch.empty(plan.out_shape, dtype=plan.data_dtype, device="cuda")
                U = plan.filter_transform(g_dev) if fx else None

                def step():
                    plan.forward(d_dev, y=y, U=U, g=None if fx else g_dev, workspace=ws)

                step()  # warm-up, untimed
                best = float("inf")
                for _ in range(repeats):
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    a.record()
                    step()
                    b.record()
                    b.synchronize()
                    best = min(best, a.elapsed_time(b) / 1e3)
        except (MemoryError, torch.cuda.OutOfMemoryError):
            rep.add(entry.label, algo, batch, None, None)
            continue
        per_instance = gflops_direct(cfg) / cfg.depth
        rep.add(entry.label, algo, batch, best * 1e3, per_instance / best)
        total_sec += best * cfg.depth
        total_gf += gflops_direct(cfg)
    if total_sec > 0:
        rep.add("TOTAL", algo, batch, total_sec * 1e3, total_gf / total_sec)
    return rep


def cmd_accuracy(suite: str = "vgg-e-accuracy", algos: Sequence[str] = ACCURACY_ALGOS,
                 precision: str = "fp32", seed: int = 0, scale: float = 1.0) -> Report:
    """Max abs error of each algorithm against the fp64 direct oracle, computed
    on the GPU (commands.py:64-92).  ``precision="fp16"`` snaps both operands to
    the binary16 grid first and keeps the oracle on the unquantized values."""
    if precision not in ("fp32", "fp16"):
        raise ValueError(f"precision must be fp32 or fp16, got {precision!r}")
    for a in algos:
        base = a.partition(":")[0]
        if a not in ACCURACY_ALGOS and a not in DIRECT_ALGOS and base not in WINOGRAD_ALGOS:
            raise ValueError(f"unknown algorithm {a!r}; known: {', '.join(ACCURACY_ALGOS)}")
    layers = get_suite(suite).scaled(scale)
    tag = "fp32" if precision == "fp32" else Precision.FP16_SIM.value
    rep = Report(columns=("layer", "algo", "precision", "max_abs_err"), seed=seed)
    for i, entry in enumerate(layers.entries):
        d, g = layer_inputs(entry.cfg, seed, i)
        oracle = direct_forward(d.astype(Precision.FP64), g.astype(Precision.FP64), entry.cfg)
        if precision == "fp16":
            d, g = quantize_fp16(d), quantize_fp16(g)
        for algo in algos:
            y = run_layer(algo, d, g, entry.cfg)
            rep.add(entry.label, algo, tag, max_abs_error(y, oracle))
    return rep
