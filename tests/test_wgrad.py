"""Weight gradient F(3x3, 2x2) (engine.py:278-328): oracle pinned to the
reference's golden outputs (CPU), host validation (CPU), and the CUDA path via
the C ABI against the oracle / fp64 direct ground truth (GPU).

Tolerances:
  * fp64: < 1e-12 abs vs fp64 direct on O(1) data (test_engine.py:253-267),
    relative 1e-10 (test_engine.py:235-242), adjoint identity rel 1e-8
    (test_engine.py:276-283).
  * fp32 (3xTF32 GEMM): < 1e-3 abs vs fp64 direct (test_engine.py:244-250) and
    <= 2e-5 * (1 + max|ref|) vs the reference's own fp32 output.
  * tf32 / bf16 / fp16: relative to max|dg|, 1e-2 / 3e-2 / 5e-3 (operand
    rounding of Uw and Vw; the tile reduction averages it down).
"""
import numpy as np
import pytest

from oracle import winograd_oracle as O


@pytest.fixture(scope="module")
def wg():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "golden_wgrad.npz")
    return np.load(path)


def _inputs(wg, i, dtype):
    N, C, H, W, K, pad = (int(v) for v in wg[f"case{i}_shape"])
    oh, ow = H + 2 * pad - 2, W + 2 * pad - 2
    d = O.fill_uniform((N, C, H, W), 500 + 2 * i, dtype=dtype)
    dy = O.fill_uniform((N, K, oh, ow), 501 + 2 * i, dtype=dtype)
    return (N, C, H, W, K, pad), d, dy


def _ncases(wg):
    return sum(1 for k in wg.files if k.endswith("_shape"))


# ----------------------------------------------------------------- CPU
def test_oracle_matches_reference_bitwise(wg):
    for i in range(_ncases(wg)):
        for dt, tag in ((np.float32, "fp32"), (np.float64, "fp64")):
            shape, d, dy = _inputs(wg, i, dt)
            out = O.winograd_grad_weights(d, dy, shape[5])
            assert np.array_equal(out, wg[f"case{i}_{tag}"]), (i, tag)
        _, d, dy = _inputs(wg, i, np.float64)
        assert np.array_equal(O.direct_grad_weights(d, dy, shape[5]), wg[f"case{i}_direct64"]), i


def test_validation_errors():
    import paper_1509_09308_b200 as wb
    T = wb.Tensor4.from_array
    cfg = wb.LayerConfig(N=1, C=1, H=6, W=6, K=1, R=2, S=2, pad=0)
    with pytest.raises(ValueError):  # test_engine.py:269-274
        wb.winograd_grad_weights(T(O.fill_uniform((1, 1, 6, 6), 10)),
                                 T(O.fill_uniform((1, 1, 5, 5), 11)), cfg)
    cfg = wb.LayerConfig(N=1, C=2, H=6, W=6, K=2, pad=1)
    d = O.fill_uniform((1, 2, 6, 6), 1)
    with pytest.raises(ValueError):  # mixed precisions
        wb.winograd_grad_weights(T(d), T(O.fill_uniform((1, 2, 6, 6), 2).astype(np.float64),
                                          wb.Precision.FP64), cfg)
    with pytest.raises(ValueError):  # dY shape
        wb.winograd_grad_weights(T(d), T(O.fill_uniform((1, 2, 5, 6), 2)), cfg)
    with pytest.raises(ValueError):  # wrong algorithm for 3x3
        wb.winograd_grad_weights(T(d), T(O.fill_uniform((1, 2, 6, 6), 2)), cfg,
                                 alg_w=wb.builtin(2, 3))
    assert wb.builtin(3, 2).alpha == 4


def test_workspace_query_host_only():
    import ctypes
    import paper_1509_09308_b200 as wb
    from paper_1509_09308_b200 import _lib
    desc = _lib.LayerDesc(64, 64, 224, 224, 64, 3, 3, 1)
    need = ctypes.c_size_t()
    assert _lib.lib.wino_wgrad_workspace(ctypes.byref(desc), 0, 64 << 20,
                                         ctypes.byref(need)) == 0
    assert 0 < need.value < (64 << 20) * 2  # chunked to the budget (+ M slices)
    desc = _lib.LayerDesc(1, 1, 6, 6, 1, 2, 2, 0)
    assert _lib.lib.wino_wgrad_workspace(ctypes.byref(desc), 0, 0, ctypes.byref(need)) == 2
    # C <= 4 (conv1.1): the small-C pass stages nothing but its M slices
    # (<= 2 per SM, 16 x K x 4 floats each), whatever the batch
    desc = _lib.LayerDesc(64, 3, 224, 224, 64, 3, 3, 1)
    for prec in (0, 1, 2, 3):
        assert _lib.lib.wino_wgrad_workspace(ctypes.byref(desc), prec, 0,
                                             ctypes.byref(need)) == 0
        assert need.value <= (2 * 148 + 1) * 16 * 64 * 4 * 4 + 1024
    # fp64 keeps the staged path
    assert _lib.lib.wino_wgrad_workspace(ctypes.byref(desc), 4, 0, ctypes.byref(need)) == 0
    assert need.value > 64 << 20
    del wb


# ----------------------------------------------------------------- GPU
def _run(wb, d, dy, shape, prec=None, counter=None):
    N, C, H, W, K, pad = shape
    cfg = wb.LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=pad)
    prc = wb.Precision.FP64 if d.dtype == np.float64 else wb.Precision.FP32
    T = wb.Tensor4.from_array
    return wb.winograd_grad_weights(T(d, prc), T(dy, prc), cfg, counter=counter, prec=prec).data


@pytest.mark.gpu
def test_golden_fp32_and_fp64(wg):
    import paper_1509_09308_b200 as wb
    for i in range(_ncases(wg)):
        shape, d, dy = _inputs(wg, i, np.float32)
        ref = wg[f"case{i}_fp32"]
        counter = wb.OpCounter()
        out = _run(wb, d, dy, shape, counter=counter)
        assert out.dtype == np.float32 and out.shape == ref.shape
        assert np.abs(out - ref).max() <= 2e-5 * (1 + np.abs(ref).max()), i
        assert O.max_abs_error(out, wg[f"case{i}_direct64"]) < 1e-3, i
        assert counter.get("mul") == int(wg[f"case{i}_mul"][0]), i
        shape, d, dy = _inputs(wg, i, np.float64)
        out = _run(wb, d, dy, shape)
        assert out.dtype == np.float64
        assert O.max_abs_error(out, wg[f"case{i}_direct64"]) < 1e-12, i
        assert O.max_abs_error(out, wg[f"case{i}_fp64"]) < 1e-12, i


@pytest.mark.gpu
def test_zero_dy_exact():
    import paper_1509_09308_b200 as wb
    d = O.fill_uniform((1, 2, 6, 6), 1)
    for prec in ("fp32", "tf32", "bf16", "fp16"):
        out = _run(wb, d, np.zeros((1, 2, 6, 6), np.float32), (1, 2, 6, 6, 2, 1), prec=prec)
        assert np.all(out == 0.0)


@pytest.mark.gpu
def test_adjoint_identity_fp64():
    import paper_1509_09308_b200 as wb
    d = O.fill_uniform((2, 3, 6, 6), 12, dtype=np.float64)
    g = O.fill_uniform((2, 3, 3, 3), 13, dtype=np.float64)
    dy = O.fill_uniform((2, 2, 6, 6), 14, dtype=np.float64)
    y = O.direct_forward(d, g, 1)
    dg = _run(wb, d, dy, (2, 3, 6, 6, 2, 1))
    assert float(np.vdot(g, dg)) == pytest.approx(float(np.vdot(y, dy)), rel=1e-8)


@pytest.mark.gpu
@pytest.mark.parametrize("prec,tol", [("tf32", 1e-2), ("bf16", 3e-2), ("fp16", 5e-3)])
def test_reduced_precision_envelope(prec, tol):
    import paper_1509_09308_b200 as wb
    d = O.fill_uniform((2, 48, 20, 18), 21)
    dy = O.fill_uniform((2, 40, 20, 18), 22)
    ref = O.direct_grad_weights(d, dy, 1)
    out = _run(wb, d, dy, (2, 48, 20, 18, 40, 1), prec=prec)
    assert O.max_abs_error(out, ref) / np.abs(ref).max() <= tol


@pytest.mark.gpu
def test_chunked_and_split_tiles():
    """A workspace budget that forces many tile chunks (and split reductions)
    sums the chunk slices to the same gradient as the fp64 ground truth."""
    import torch
    import paper_1509_09308_b200 as wb
    cfg = wb.LayerConfig(N=3, C=64, H=28, W=26, K=96, pad=1)
    dn = O.fill_uniform((3, 64, 28, 26), 31)
    yn = O.fill_uniform((3, 96, 28, 26), 32)
    ref = O.direct_grad_weights(dn, yn, 1)
    d, dy = torch.from_numpy(dn).cuda(), torch.from_numpy(yn).cuda()
    a = wb.grad_weights_device(d, dy, cfg, "fp32").cpu().numpy()
    b = wb.grad_weights_device(d, dy, cfg, "fp32", workspace_limit=1 << 20).cpu().numpy()
    for out in (a, b):
        assert O.max_abs_error(out, ref) < 1e-3
    assert np.abs(a - b).max() <= 1e-5 * (1 + np.abs(ref).max())


@pytest.mark.gpu
@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("tf32", 1e-2), ("bf16", 3e-2),
                                      ("fp16", 5e-3)])
def test_small_c(prec, tol, monkeypatch):
    """conv1.1-like shape (C = 3, ragged tile count): the CUDA-core small-C
    pass and the tensor-core GEMM path (many tile splits, kept or folded
    slices) all match the fp64 ground truth."""
    import torch
    import paper_1509_09308_b200 as wb
    cfg = wb.LayerConfig(N=2, C=3, H=63, W=61, K=70, pad=1)
    dn = O.fill_uniform((2, 3, 63, 61), 41)
    yn = O.fill_uniform((2, 70, 63, 61), 42)
    ref = O.direct_grad_weights(dn, yn, 1)
    d, dy = torch.from_numpy(dn).cuda(), torch.from_numpy(yn).cuda()
    scale = np.abs(ref).max()
    small = wb.grad_weights_device(d, dy, cfg, prec).cpu().numpy()
    assert O.max_abs_error(small, ref) / scale <= tol
    monkeypatch.setenv("WINO_NO_WGRAD_SMALLC", "1")
    gemm = wb.grad_weights_device(d, dy, cfg, prec).cpu().numpy()
    fold = wb.grad_weights_device(d, dy, cfg, prec, workspace_limit=1 << 20).cpu().numpy()
    for out in (gemm, fold):
        assert O.max_abs_error(out, ref) / scale <= tol
    assert np.abs(gemm - fold).max() <= 1e-5 * (1 + scale)
