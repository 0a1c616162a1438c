"""Generate golden fixtures from the REAL reference package (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Every array in it is an output of
``winoconv`` itself (the reference, imported read-only), so the oracle and the
CUDA path are pinned to the reference's arithmetic, not to our restatement.
The GPU box never runs this script (``/root/reference`` does not exist there);
it only reads the committed .npz.
"""
from __future__ import annotations

import os
import random
import sys

import numpy as np

sys.path.insert(0, os.environ.get("WINO_REF_SRC", "/root/reference/pkg/src"))

from winoconv.counters import OpCounter  # noqa: E402
from winoconv.direct import LayerConfig, direct_forward  # noqa: E402
from winoconv.engine import (FilterCache, TileGrid, multiply_stage_flops,  # noqa: E402
                             tile_count, transform_filters, winograd_forward)
from winoconv.tensors import (Precision, Tensor4, _splitmix64_unit_doubles,  # noqa: E402
                              fill_uniform, quantize_fp16)
from winoconv.winograd import builtin  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

# Small whole-layer cases: (N, C, H, W, K, pad); include ragged edges, pad 0/1,
# single channel, C not a multiple of anything.
LAYER_CASES = [
    (1, 1, 6, 6, 1, 0),
    (1, 1, 5, 5, 1, 0),
    (1, 1, 7, 9, 2, 1),
    (3, 4, 11, 5, 3, 1),
    (2, 8, 12, 12, 4, 0),
    (1, 16, 15, 14, 8, 1),
    (2, 3, 9, 9, 5, 1),
    (1, 33, 13, 10, 17, 1),
    (1, 8, 14, 14, 8, 1),
    (1, 64, 20, 20, 64, 1),
]


def rand(shape, seed, prec=Precision.FP32):
    return fill_uniform(Tensor4.zeros(shape, precision=prec), seed, -1.0, 1.0)


def main() -> None:
    g = {}
    # SplitMix64 streams and fills (tensors.py:122-153)
    for s in (0, 1, 7, 12345, 2**63 + 5, 2**64 - 1):
        g[f"sm64_{s}"] = _splitmix64_unit_doubles(257, s)
    g["fill_f32_s3"] = rand((2, 3, 5, 7), 3).data.copy()
    g["fill_f64_s4"] = rand((1, 2, 3, 4), 4, Precision.FP64).data.copy()
    g["fill_f32_lohi"] = fill_uniform(Tensor4.zeros((1, 1, 4, 64)), 9, -0.5, 2.0).data.copy()
    g["fp16_q"] = quantize_fp16(rand((1, 2, 8, 8), 11)).data.copy()

    # lowered matrices (engine.py:98-101)
    for (m, r) in ((2, 3), (4, 3), (3, 2)):
        alg = builtin(m, r)
        for dt in (np.float32, np.float64):
            tag = np.dtype(dt).name
            g[f"BT_{m}{r}_{tag}"] = alg.BT.to_array(dt)
            g[f"G_{m}{r}_{tag}"] = alg.G.to_array(dt)
            g[f"AT_{m}{r}_{tag}"] = alg.AT.to_array(dt)

    # tile grids (engine.py:40-95)
    grid_cases = [(2, 1, 13, 11, 1, 1, 2), (2, 1, 8, 8, 1, 0, 2), (1, 1, 224, 224, 1, 1, 2),
                  (1, 1, 14, 14, 1, 1, 4), (32, 1, 28, 28, 1, 1, 2), (3, 2, 17, 9, 4, 1, 4)]
    rows = []
    for (N, C, H, W, K, pad, m) in grid_cases:
        cfg = LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=pad)
        grid = TileGrid.for_layer(cfg, m, 3)
        samples = sorted({0, 1, grid.P // 2, grid.P - 1})
        for b in samples:
            n, ty, tx = grid.index(b)
            oy, ox = grid.origin(b)
            rows.append([N, C, H, W, K, pad, m, grid.tiles_h, grid.tiles_w, grid.P,
                         tile_count(cfg, m), multiply_stage_flops(cfg, m), b, n, ty, tx, oy, ox])
    g["tile_grid"] = np.array(rows, dtype=np.int64)

    # whole-layer forward, both algorithms, fp32 and fp64, plus the fp64 oracle
    for i, (N, C, H, W, K, pad) in enumerate(LAYER_CASES):
        cfg = LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=pad)
        d = rand((N, C, H, W), 100 + 2 * i)
        w = rand((K, C, 3, 3), 101 + 2 * i)
        g[f"case{i}_shape"] = np.array([N, C, H, W, K, pad], dtype=np.int64)
        g[f"case{i}_direct64"] = direct_forward(d.astype(Precision.FP64),
                                                w.astype(Precision.FP64), cfg).data.copy()
        for m in (2, 4):
            alg = builtin(m, 3)
            c = OpCounter()
            y = winograd_forward(d, w, cfg, alg, counter=c)
            g[f"case{i}_f{m}_fp32"] = y.data.copy()
            g[f"case{i}_f{m}_mul"] = np.array(c.get("mul"), dtype=np.int64)
            y64 = winograd_forward(d.astype(Precision.FP64), w.astype(Precision.FP64), cfg, alg)
            g[f"case{i}_f{m}_fp64"] = y64.data.copy()
            cache = FilterCache()
            yfx = winograd_forward(d, w, cfg, alg, cache_filters=True, cache=cache)
            assert np.array_equal(yfx.data, y.data)
            if K * C <= 512:
                g[f"case{i}_f{m}_U"] = transform_filters(w, alg)
        dq, wq = quantize_fp16(d), quantize_fp16(w)
        g[f"case{i}_f4_fp16sim"] = winograd_forward(dq, wq, cfg, builtin(4, 3)).data.copy()

    # config 1 (N=1 C=K=64 56x56 pad=1): strided sample + summary of the reference output
    cfg = LayerConfig(N=1, C=64, H=56, W=56, K=64, pad=1)
    d = fill_uniform(Tensor4.zeros((1, 64, 56, 56)), 0, -1.0, 1.0)
    w = fill_uniform(Tensor4.zeros((64, 64, 3, 3)), 1, -1.0, 1.0)
    for m in (2, 4):
        y = winograd_forward(d, w, cfg, builtin(m, 3)).data
        g[f"cfg1_f{m}_sample"] = y.reshape(-1)[::37].copy()
        g[f"cfg1_f{m}_sum"] = np.array([y.astype(np.float64).sum(),
                                        np.abs(y.astype(np.float64)).sum()])

    # the acceptance sweep's shapes (test_acceptance.py:120-142), seed 55
    rng = random.Random(55)
    shapes = []
    for _ in range(200):
        shapes.append([rng.randint(1, 4), rng.randint(1, 32), rng.randint(3, 40),
                       rng.randint(3, 40), rng.randint(1, 32), rng.choice((0, 1))])
    g["sweep55_shapes"] = np.array(shapes, dtype=np.int64)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e3:.0f} kB")


if __name__ == "__main__":
    main()
