"""Golden fixtures for the weight gradient, from the REAL reference package.

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_wgrad.py

Writes tests/golden/golden_wgrad.npz: for each case, the inputs' seeds and the
reference's own ``winograd_grad_weights`` output (F(3x3,2x2), engine.py:278-328)
at fp32 and fp64, plus its ``direct_grad_weights`` fp64 ground truth
(direct.py:149-177).  Inputs come from ``fill_uniform`` (SplitMix64), which the
oracle reproduces bit for bit, so the fixture only stores outputs.
The GPU box never runs this script; it reads the committed .npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("WINO_REF_SRC", "/root/reference/pkg/src"))

from winoconv.counters import OpCounter  # noqa: E402
from winoconv.direct import LayerConfig, direct_grad_weights  # noqa: E402
from winoconv.engine import winograd_grad_weights  # noqa: E402
from winoconv.tensors import Precision, Tensor4, fill_uniform  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_wgrad.npz")

# (N, C, H, W, K, pad): the reference tests' shapes (test_engine.py:226-283)
# plus ragged / multi-image / wider cases.
CASES = [
    (1, 2, 6, 6, 2, 1),
    (1, 1, 6, 6, 1, 1),
    (2, 4, 8, 8, 4, 1),
    (1, 2, 7, 5, 3, 1),
    (1, 1, 8, 8, 1, 0),
    (2, 3, 6, 6, 2, 1),
    (1, 16, 15, 14, 8, 1),
    (3, 33, 9, 11, 20, 1),
    (2, 24, 12, 10, 40, 0),
]


def main() -> None:
    out = {}
    for i, (N, C, H, W, K, pad) in enumerate(CASES):
        cfg = LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=pad)
        out[f"case{i}_shape"] = np.array([N, C, H, W, K, pad], dtype=np.int64)
        for prec, tag in ((Precision.FP32, "fp32"), (Precision.FP64, "fp64")):
            d = fill_uniform(Tensor4.zeros((N, C, H, W), precision=prec), 500 + 2 * i, -1.0, 1.0)
            dy = fill_uniform(Tensor4.zeros((N, K, cfg.out_h, cfg.out_w), precision=prec),
                              501 + 2 * i, -1.0, 1.0)
            counter = OpCounter()
            dg = winograd_grad_weights(d, dy, cfg, counter=counter)
            out[f"case{i}_{tag}"] = np.asarray(dg.data)
            out[f"case{i}_mul"] = np.array([counter.get("mul")], dtype=np.int64)
            if tag == "fp64":
                out[f"case{i}_direct64"] = np.asarray(direct_grad_weights(d, dy, cfg).data)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays")


if __name__ == "__main__":
    main()
