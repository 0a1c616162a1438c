"""Full-size VGG-E fixtures from the REAL reference package (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_vgg.py

For every VGG-E conv shape (suites.py:68-78) at N=1, with the inputs
``cmd_bench`` / ``cmd_accuracy`` generate (``_layer_inputs``, seed 0,
commands.py:54-61), this records the reference's own ``winograd_forward``
output for F(2x2,3x3) and F(4x4,3x3) at fp32, and F(4x4,3x3) on fp16-sim
operands (the ``cmd_accuracy --precision fp16`` path, commands.py:64-92):

* a strided sample of y (every ``stride``-th element of the flat NCHW output),
* fp64 sum and abs-sum of the whole y, and max |y|,
* the reference's max-abs error against its own fp64 direct convolution
  (the accuracy envelope the GPU gates are stated against).

Inputs are SplitMix64 fills, so image 0 of any batch N made with the same seed
equals this N=1 image (the fill is one flat stream): the same fixtures pin image
0 of the N = 8 / 16 / 32 / 64 plans the bench times.  The GPU box never runs this
script; it reads the committed tests/golden/golden_vgg.npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("WINO_REF_SRC", "/root/reference/pkg/src"))

from winoconv.commands import _layer_inputs  # noqa: E402
from winoconv.direct import LayerConfig, direct_forward  # noqa: E402
from winoconv.engine import winograd_forward  # noqa: E402
from winoconv.suites import get_suite  # noqa: E402
from winoconv.tensors import Precision, quantize_fp16  # noqa: E402
from winoconv.winograd import builtin  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_vgg.npz")
SAMPLES = 4096


def stride_for(size: int) -> int:
    s = max(1, size // SAMPLES)
    return s | 1  # odd: the sample walks across rows, columns and filters


def summary(g: dict, key: str, y: np.ndarray, oracle: np.ndarray) -> None:
    y64 = y.astype(np.float64)
    st = stride_for(y.size)
    g[f"{key}_stride"] = np.array(st, dtype=np.int64)
    g[f"{key}_sample"] = y.reshape(-1)[::st].copy()
    g[f"{key}_sums"] = np.array([y64.sum(), np.abs(y64).sum(), np.abs(y64).max(),
                                 float(np.abs(y64 - oracle.astype(np.float64)).max())])


def main() -> None:
    g = {}
    suite = get_suite("vgg-e")
    rows = []
    for i, entry in enumerate(suite.entries):
        c = entry.cfg
        cfg = LayerConfig(N=1, C=c.C, H=c.H, W=c.W, K=c.K, pad=c.pad)
        rows.append([i, c.C, c.H, c.W, c.K, c.pad])
        d, w = _layer_inputs(cfg, 0, i)
        oracle = direct_forward(d.astype(Precision.FP64), w.astype(Precision.FP64), cfg).data
        for m in (2, 4):
            y = winograd_forward(d, w, cfg, builtin(m, 3)).data
            summary(g, f"L{i}_f{m}_fp32", y, oracle)
        dq, wq = quantize_fp16(d), quantize_fp16(w)
        y = winograd_forward(dq, wq, cfg, builtin(4, 3)).data
        summary(g, f"L{i}_f4_fp16sim", y, oracle)
        print(f"layer {i} ({entry.label}) done", flush=True)
    g["layers"] = np.array(rows, dtype=np.int64)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e3:.0f} kB")


if __name__ == "__main__":
    main()
