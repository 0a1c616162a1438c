"""GPU direct correlation (``wino_direct_forward``) and the accuracy harness
(``cmd_accuracy``) against fixtures made by the reference itself
(tests/golden/make_golden_direct.py).  The direct kernel accumulates in the
reference's order with a rounded multiply and a rounded add, so the gates here
are bitwise."""
import os

import numpy as np
import pytest

from oracle import winograd_oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def wb():
    import paper_1509_09308_b200 as wb
    return wb


@pytest.fixture(scope="module")
def gd():
    return np.load(os.path.join(HERE, "golden", "golden_direct.npz"))


def test_direct_bitwise_vs_reference(wb, golden, gd):
    for i in range(10):
        N, C, H, W, K, pad = (int(v) for v in golden[f"case{i}_shape"])
        cfg = wb.LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=pad)
        d = wb.Tensor4.from_array(O.fill_uniform((N, C, H, W), 100 + 2 * i), wb.Precision.FP32)
        g = wb.Tensor4.from_array(O.fill_uniform((K, C, 3, 3), 101 + 2 * i), wb.Precision.FP32)
        y32 = wb.run_layer("direct-fp32", d, g, cfg)
        assert y32.precision is wb.Precision.FP32
        assert np.array_equal(y32.data, gd[f"case{i}_direct32"]), i
        y64 = wb.direct_forward(d, g, cfg)  # fp64 accumulator on fp32 data
        assert np.array_equal(y64.data, golden[f"case{i}_direct64"]), i
        d64, g64 = d.astype(wb.Precision.FP64), g.astype(wb.Precision.FP64)
        assert np.array_equal(wb.run_layer("direct", d64, g64, cfg).data,
                              gd[f"case{i}_direct64f64"]), i


def test_direct_counter_and_errors(wb):
    cfg = wb.LayerConfig(N=2, C=3, H=7, W=5, K=4, pad=1)
    d = wb.Tensor4.from_array(O.fill_uniform((2, 3, 7, 5), 1), wb.Precision.FP32)
    g = wb.Tensor4.from_array(O.fill_uniform((4, 3, 3, 3), 2), wb.Precision.FP32)
    c = wb.OpCounter()
    wb.direct_forward(d, g, cfg, counter=c)
    # brute force: one multiply per in-image tap per output
    taps = 0
    for x in range(cfg.out_h):
        for y in range(cfg.out_w):
            for u in range(3):
                for v in range(3):
                    if 0 <= x + u - 1 < 7 and 0 <= y + v - 1 < 5:
                        taps += 1
    assert c.get("mul") == 2 * 4 * 3 * taps
    with pytest.raises(ValueError):
        wb.direct_forward(d, g, cfg, accum=wb.Precision.FP16_SIM)


def test_cmd_accuracy_matches_reference(wb, gd):
    """direct-fp32 rows of the GPU accuracy report equal the reference's
    cmd_accuracy rows (scale 1/8 VGG-E accuracy suite); the Winograd rows stay
    inside the reference's fp32 gates (test_engine.py:97-112)."""
    rep = wb.cmd_accuracy(algos=("direct-fp32", "f2x2", "f4x4"), scale=0.125)
    rows = {(r[0], r[1]): r[3] for r in rep.rows}
    for lbl, ref in zip(gd["acc_labels"], gd["acc_rows"]):
        assert rows[(str(lbl), "direct-fp32")] == ref, lbl
        assert rows[(str(lbl), "f2x2")] < 5e-4 and rows[(str(lbl), "f4x4")] < 5e-3, lbl


def test_fft_layer_vs_reference(wb, golden, gd):
    """The FFT comparison algorithm (hand-written fp64 DFT + complex GEMM kernels, the reference's
    tiling and fp64 transform arithmetic) against the reference's own outputs:
    fp64 within 1e-12 (relative to max|y|), fp32 within 1 fp32 rounding of the
    final cast (2^-23 relative); counters equal."""
    for i in range(10):
        N, C, H, W, K, pad = (int(v) for v in golden[f"case{i}_shape"])
        cfg = wb.LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=pad)
        d = wb.Tensor4.from_array(O.fill_uniform((N, C, H, W), 100 + 2 * i), wb.Precision.FP32)
        g = wb.Tensor4.from_array(O.fill_uniform((K, C, 3, 3), 101 + 2 * i), wb.Precision.FP32)
        cnt = wb.OpCounter()
        y = wb.run_layer("fft", d, g, cfg, counter=cnt)
        ref = gd[f"case{i}_fft32"]
        assert y.data.dtype == np.float32 and y.data.shape == ref.shape
        assert np.abs(y.data - ref).max() <= 2 ** -23 * (1 + np.abs(ref).max()), i
        assert [cnt.get("cmul"), cnt.get("mul")] == list(gd[f"case{i}_fft_counts"]), i
        y64 = wb.run_layer("fft", d.astype(wb.Precision.FP64), g.astype(wb.Precision.FP64), cfg)
        ref64 = gd[f"case{i}_fft64"]
        assert np.abs(y64.data - ref64).max() <= 1e-12 * (1 + np.abs(ref64).max()), i
