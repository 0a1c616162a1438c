"""Golden fixtures for the direct-correlation, FFT and accuracy paths, made by
the REAL reference package (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_direct.py

Writes tests/golden/golden_direct.npz:
  * case{i}_direct32 -- winoconv.direct.direct_forward(d, g, cfg, accum=FP32) on the
    golden.npz layer cases (seeds 100+2i / 101+2i), and case{i}_direct64f64 on
    fp64 inputs;
  * case{i}_fft32 / case{i}_fft64 and case{i}_fft_counts (cmul, mul) --
    winoconv.fftconv.fft_forward_layer(tile=8) on fp32 / fp64 inputs;
  * acc_rows -- winoconv.commands.cmd_accuracy(algos=("direct-fp32",),
    scale=0.125) max_abs_err per layer (direct-fp32 vs the fp64 oracle).
The GPU box only reads the committed .npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("WINO_REF_SRC", "/root/reference/pkg/src"))

from winoconv.commands import cmd_accuracy  # noqa: E402
from winoconv.counters import OpCounter  # noqa: E402
from winoconv.direct import LayerConfig, direct_forward  # noqa: E402
from winoconv.fftconv import fft_forward_layer  # noqa: E402
from winoconv.tensors import Precision, Tensor4, fill_uniform  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import LAYER_CASES  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_direct.npz")


def main() -> None:
    g = {}
    for i, (N, C, H, W, K, pad) in enumerate(LAYER_CASES):
        cfg = LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=pad)
        d = fill_uniform(Tensor4.zeros((N, C, H, W)), 100 + 2 * i, -1.0, 1.0)
        w = fill_uniform(Tensor4.zeros((K, C, 3, 3)), 101 + 2 * i, -1.0, 1.0)
        g[f"case{i}_direct32"] = direct_forward(d, w, cfg, accum=Precision.FP32).data
        g[f"case{i}_direct64f64"] = direct_forward(d.astype(Precision.FP64),
                                                   w.astype(Precision.FP64), cfg).data
        cnt = OpCounter()
        g[f"case{i}_fft32"] = fft_forward_layer(d, w, cfg, tile=8, counter=cnt).data
        g[f"case{i}_fft_counts"] = np.array([cnt.get("cmul"), cnt.get("mul")], dtype=np.int64)
        g[f"case{i}_fft64"] = fft_forward_layer(d.astype(Precision.FP64),
                                                w.astype(Precision.FP64), cfg, tile=8).data
    rep = cmd_accuracy(algos=("direct-fp32",), scale=0.125)
    g["acc_labels"] = np.array([r[0] for r in rep.rows])
    g["acc_rows"] = np.array([r[3] for r in rep.rows], dtype=np.float64)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays")


if __name__ == "__main__":
    main()
