"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden outputs on identical SplitMix64 inputs.

Tolerances (max-abs, stated per F(m,r) and GEMM precision):
  * vs fp64 direct conv: the reference's own gates, F2 < 5e-4, F4 < 5e-3 for
    the fp32 (3xTF32) path (test_engine.py:97-112); fp64 < 1e-12
    (test_engine.py:114-119).
  * vs the reference's fp32 Winograd output: |diff| <= 2e-5 * (1 + max|y|)
    for fp32 (both are fp32-accurate; only summation order differs).
  * reduced-precision GEMMs, relative to max|y|: tf32 <= 1e-2 (F2) / 4e-2 (F4);
    fp16 <= 4e-3 / 2.5e-2; bf16 <= 2e-2 / 1.5e-1  (operand rounding of U and V,
    plus the 16-bit staging of M).
"""
import numpy as np
import pytest

from oracle import winograd_oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = {("tf32", 2): 1e-2, ("tf32", 4): 4e-2, ("fp16", 2): 4e-3, ("fp16", 4): 2.5e-2,
           ("bf16", 2): 2e-2, ("bf16", 4): 1.5e-1}


@pytest.fixture(scope="module")
def wb():
    import paper_1509_09308_b200 as wb
    return wb


# The three forward paths of the C planner (WINO_PATH, read at plan creation):
# staged (input transform -> GEMM -> output transform), fused (one kernel),
# hybrid (staged input transform + fused GEMM/inverse transform).
PATHS = ["staged", "fused", "hybrid"]


@pytest.fixture(params=PATHS)
def path(request, monkeypatch):
    monkeypatch.setenv("WINO_PATH", request.param)
    return request.param


def _run(wb, d, g, pad, m, prec=None, fx=False, cache=None):
    cfg = wb.LayerConfig(N=d.shape[0], C=d.shape[1], H=d.shape[2], W=d.shape[3], K=g.shape[0],
                         pad=pad)
    prc = wb.Precision.FP64 if d.dtype == np.float64 else wb.Precision.FP32
    return wb.winograd_forward(wb.Tensor4.from_array(d, prc), wb.Tensor4.from_array(g, prc), cfg,
                               wb.builtin(m, 3), cache_filters=fx, cache=cache, prec=prec).data


@pytest.mark.parametrize("m", [2, 4])
def test_golden_cases_fp32(wb, golden, m, path):
    for i in range(10):
        N, C, H, W, K, pad = (int(v) for v in golden[f"case{i}_shape"])
        d = O.fill_uniform((N, C, H, W), 100 + 2 * i)
        g = O.fill_uniform((K, C, 3, 3), 101 + 2 * i)
        y = _run(wb, d, g, pad, m)
        ref = golden[f"case{i}_f{m}_fp32"]
        direct = golden[f"case{i}_direct64"]
        assert y.shape == ref.shape
        scale = 1.0 + np.abs(ref).max()
        assert np.abs(y - ref).max() <= 2e-5 * scale, (i, np.abs(y - ref).max())
        assert O.max_abs_error(y, direct) < (5e-4 if m == 2 else 5e-3), i


@pytest.mark.parametrize("m", [2, 4])
def test_golden_cases_fp64(wb, golden, m):
    for i in range(10):
        N, C, H, W, K, pad = (int(v) for v in golden[f"case{i}_shape"])
        d = O.fill_uniform((N, C, H, W), 100 + 2 * i).astype(np.float64)
        g = O.fill_uniform((K, C, 3, 3), 101 + 2 * i).astype(np.float64)
        y = _run(wb, d, g, pad, m)
        assert y.dtype == np.float64
        assert O.max_abs_error(y, golden[f"case{i}_direct64"]) < 1e-12, i
        assert O.max_abs_error(y, golden[f"case{i}_f{m}_fp64"]) < 1e-12, i


@pytest.mark.parametrize("m", [2, 4])
@pytest.mark.parametrize("prec", ["tf32", "bf16", "fp16"])
def test_reduced_precision_envelope(wb, golden, m, prec, path):
    for i in (3, 5, 7, 9):
        N, C, H, W, K, pad = (int(v) for v in golden[f"case{i}_shape"])
        d = O.fill_uniform((N, C, H, W), 100 + 2 * i)
        g = O.fill_uniform((K, C, 3, 3), 101 + 2 * i)
        y = _run(wb, d, g, pad, m, prec=prec)
        ref = golden[f"case{i}_direct64"]
        err = O.max_abs_error(y, ref) / np.abs(ref).max()
        assert err <= REL_TOL[(prec, m)], (i, err)


def test_config1_against_reference(wb, golden):
    """Config 1 (N=1 C=K=64 56x56 pad=1) vs the reference's recorded output."""
    d = O.fill_uniform((1, 64, 56, 56), 0)
    g = O.fill_uniform((64, 64, 3, 3), 1)
    for m in (2, 4):
        y = _run(wb, d, g, 1, m)
        samp = y.reshape(-1)[::37]
        ref = golden[f"cfg1_f{m}_sample"]
        assert np.abs(samp - ref).max() <= 2e-5 * (1 + np.abs(ref).max())
        s = golden[f"cfg1_f{m}_sum"]
        assert abs(y.astype(np.float64).sum() - s[0]) <= 1e-6 * s[1]


def test_zero_filters_exact(wb, path):
    d = O.fill_uniform((1, 2, 6, 6), 1)
    g = np.zeros((2, 2, 3, 3), np.float32)
    for m in (2, 4):
        for prec in ("fp32", "tf32", "bf16", "fp16"):
            assert np.all(_run(wb, d, g, 1, m, prec=prec) == 0.0)


def test_impulse_filter_copies_input(wb, path):
    """A centred delta filter reproduces the input: any tile-indexing or
    padding slip would show as O(1) errors.  Exact for F(2x2) (all transform
    constants are dyadic); F(4x4)'s 1/6, 1/12, 1/24 round in fp32."""
    d = O.fill_uniform((2, 3, 13, 11), 5)
    g = np.zeros((3, 3, 3, 3), np.float32)
    for k in range(3):
        g[k, k, 1, 1] = 1.0
    for m in (2, 4):
        y = _run(wb, d, g, 1, m)
        np.testing.assert_allclose(y, d, atol=(1e-6 if m == 2 else 1e-5), rtol=0)


def test_impulse_f2_bit_exact_all_precisions(wb, path):
    """F(2x2)'s transform constants are dyadic, so with inputs on a coarse
    dyadic grid (k/16, |k| <= 16: every sum and product of the transforms is
    exact in fp32 and in every operand format, bf16 included) a centred delta
    filter must copy the input BIT FOR BIT through the whole pipeline -- tile
    indexing, virtual padding, ragged edges, split-C and the inverse transform."""
    d = (np.round(O.fill_uniform((2, 5, 13, 11), 6) * 16.0) / 16.0).astype(np.float32)
    g = np.zeros((5, 5, 3, 3), np.float32)
    for k in range(5):
        g[k, k, 1, 1] = 1.0
    for prec in ("fp32", "tf32", "fp16", "bf16"):
        y = _run(wb, d, g, 1, 2, prec=prec)
        assert np.array_equal(y, d), (prec, float(np.abs(y - d).max()))


def test_fx_cache_bitwise_and_counts(wb):
    d = O.fill_uniform((1, 8, 9, 9), 9)
    g = O.fill_uniform((4, 8, 3, 3), 10)
    cache = wb.FilterCache()
    a = _run(wb, d, g, 1, 4, fx=True, cache=cache)
    b = _run(wb, d, g, 1, 4, fx=True, cache=cache)
    c = _run(wb, d, g, 1, 4)
    assert cache.misses == 1 and cache.hits == 1 and len(cache) == 1
    assert np.array_equal(a, b) and np.array_equal(a, c)
    assert cache.workspace_scalars() == 36 * 4 * 8


def test_bitwise_deterministic(wb, path):
    d = O.fill_uniform((1, 8, 9, 9), 9)
    g = O.fill_uniform((4, 8, 3, 3), 10)
    for prec in ("fp32", "bf16"):
        assert np.array_equal(_run(wb, d, g, 1, 2, prec=prec), _run(wb, d, g, 1, 2, prec=prec))


def test_chunked_planner_matches_single_chunk(wb, monkeypatch):
    """Workspace-limited plans (many row chunks) give bit-identical outputs."""
    import torch
    monkeypatch.setenv("WINO_PATH", "staged")
    cfg = wb.LayerConfig(N=2, C=16, H=30, W=22, K=24, pad=1)
    d = torch.from_numpy(O.fill_uniform((2, 16, 30, 22), 3)).cuda()
    g = torch.from_numpy(O.fill_uniform((24, 16, 3, 3), 4)).cuda()
    for m in (2, 4):
        big = wb.WinogradPlan(cfg, m, "fp32")
        small = wb.WinogradPlan(cfg, m, "fp32", workspace_limit=64 * 1024)
        assert big.info["num_chunks"] == 1 and small.info["num_chunks"] > 3
        ya = big.forward(d, g=g)
        yb = small.forward(d, g=g)
        torch.cuda.synchronize()
        assert torch.equal(ya, yb)


_SWEEP_REF = {}


def _sweep_case(golden, i):
    if i not in _SWEEP_REF:
        N, C, H, W, K, pad = (int(v) for v in golden["sweep55_shapes"][i])
        d = O.fill_uniform((N, C, H, W), 1000 + 2 * i)
        g = O.fill_uniform((K, C, 3, 3), 1001 + 2 * i)
        _SWEEP_REF[i] = (d, g, pad, O.direct_forward(d, g, pad))
    return _SWEEP_REF[i]


# relative-to-max|y| gates of the low-precision GEMMs on the sweep (measured
# envelope x ~2: the sweep's C <= 32 keeps errors below the VGG-E ones)
SWEEP_REL = {("tf32", 2): 2e-3, ("tf32", 4): 2e-2, ("fp16", 2): 2e-3, ("fp16", 4): 2e-2,
             ("bf16", 2): 1.5e-2, ("bf16", 4): 1.5e-1}


@pytest.mark.parametrize("prec", ["fp32", "tf32", "fp16", "bf16"])
def test_random_shape_sweep(wb, golden, path, prec):
    """All 200 shapes of the reference's acceptance sweep (seed 55,
    test_acceptance.py:120-142) in every GEMM precision: fp32 (3xTF32) at the
    reference's gates (F2 < 5e-4, F4 < 5e-3 vs fp64 direct), the others
    relative to max|y|."""
    worst = {2: 0.0, 4: 0.0}
    for i in range(len(golden["sweep55_shapes"])):
        d, g, pad, ref = _sweep_case(golden, i)
        scale = max(1.0, float(np.abs(ref).max()))
        for m in (2, 4):
            e = O.max_abs_error(_run(wb, d, g, pad, m, prec=prec), ref)
            worst[m] = max(worst[m], e if prec == "fp32" else e / scale)
    if prec == "fp32":
        assert worst[2] < 5e-4 and worst[4] < 5e-3, worst
    else:
        assert worst[2] <= SWEEP_REL[(prec, 2)] and worst[4] <= SWEEP_REL[(prec, 4)], worst


def test_grad_inputs_matches_oracle(wb):
    d = O.fill_uniform((1, 4, 10, 10), 7)
    g = O.fill_uniform((6, 4, 3, 3), 8)
    dy = O.fill_uniform((1, 6, 10, 10), 9)
    cfg = wb.LayerConfig(N=1, C=4, H=10, W=10, K=6, pad=1)
    T = wb.Tensor4.from_array
    out = wb.winograd_grad_inputs(T(dy), T(g), cfg, wb.builtin(4, 3)).data
    flipped = np.ascontiguousarray(g[:, :, ::-1, ::-1].transpose(1, 0, 2, 3))
    ref = O.direct_forward(dy, flipped, 1)
    assert O.max_abs_error(out, ref) < 5e-3


@pytest.mark.parametrize("m,prec", [(2, "fp32"), (4, "fp32"), (4, "bf16"), (2, "tf32")])
def test_split_c_small_p_layer(wb, m, prec, path):
    """conv5-like small-P layer: the planner splits the channel reduction across
    CTAs (staged: M slices summed by the output transform; fused/hybrid: partial
    y slices summed in split order); the result must re-assemble exactly."""
    import torch
    cfg = wb.LayerConfig(N=1, C=512, H=14, W=14, K=128, pad=1)
    plan = wb.WinogradPlan(cfg, m, prec)
    assert plan.info["fused"] == PATHS.index(path)
    if path == "staged":
        assert plan.info["gemm_splits"] > 1
    else:
        assert plan.info["fused_splits"] > 1
    d = O.fill_uniform((1, 512, 14, 14), 31)
    g = O.fill_uniform((128, 512, 3, 3), 32)
    y = plan.forward(torch.from_numpy(d).cuda(), g=torch.from_numpy(g).cuda()).cpu().numpy()
    ref = O.direct_forward(d, g, 1)
    if prec == "fp32":
        assert O.max_abs_error(y, ref) < (5e-4 if m == 2 else 5e-3)
        yo = O.winograd_forward(d, g, m, 1)
        assert np.abs(y - yo).max() <= 2e-5 * (1 + np.abs(yo).max())
    else:
        assert O.max_abs_error(y, ref) / np.abs(ref).max() <= REL_TOL[(prec, m)]


def test_hybrid_chunked_matches_oracle(wb, monkeypatch):
    """Hybrid path with a workspace that forces many V row chunks (the fused
    kernel's tile offset p0 and the chunk-local V map): same result as one chunk
    up to summation order, and within the fp32 gate of the reference."""
    import torch
    monkeypatch.setenv("WINO_PATH", "hybrid")
    cfg = wb.LayerConfig(N=2, C=40, H=30, W=22, K=24, pad=1)
    dn = O.fill_uniform((2, 40, 30, 22), 13)
    gn = O.fill_uniform((24, 40, 3, 3), 14)
    d, g = torch.from_numpy(dn).cuda(), torch.from_numpy(gn).cuda()
    ref = O.direct_forward(dn, gn, 1)
    for m in (2, 4):
        small = wb.WinogradPlan(cfg, m, "fp32", workspace_limit=256 * 1024)
        assert small.info["fused"] == 2 and small.info["num_chunks"] > 2
        y = small.forward(d, g=g).cpu().numpy()
        assert O.max_abs_error(y, ref) < (5e-4 if m == 2 else 5e-3)
        yo = O.winograd_forward(dn, gn, m, 1)
        assert np.abs(y - yo).max() <= 2e-5 * (1 + np.abs(yo).max())


@pytest.mark.parametrize("force", [False, True])
def test_plane_staged_input_transform(wb, monkeypatch, force):
    """Small planes with rows that are not 16-byte aligned (VGG conv5: 14 x 14)
    take the whole-plane staged input transform; forced on a row-chunked plan it
    must also handle chunks that start and end inside an image."""
    import torch
    monkeypatch.setenv("WINO_PATH", "staged")
    if force:
        monkeypatch.setenv("WINO_FORCE_PLANE_INPUT", "1")
    N, C, H, W, K = (80, 72, 10, 10, 16) if not force else (6, 72, 10, 10, 16)
    cfg = wb.LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=1)
    dn = O.fill_uniform((N, C, H, W), 41)
    gn = O.fill_uniform((K, C, 3, 3), 42)
    d, g = torch.from_numpy(dn).cuda(), torch.from_numpy(gn).cuda()
    ref = O.direct_forward(dn, gn, 1)
    for m in (2, 4):
        plan = wb.WinogradPlan(cfg, m, "fp32", workspace_limit=(96 * 1024 if force else 0))
        if force:
            assert plan.info["num_chunks"] > 2
        y = plan.forward(d, g=g).cpu().numpy()
        assert O.max_abs_error(y, ref) < (5e-4 if m == 2 else 5e-3)
        yo = O.winograd_forward(dn, gn, m, 1)
        assert np.abs(y - yo).max() <= 2e-5 * (1 + np.abs(yo).max())
        yb = wb.WinogradPlan(cfg, m, "bf16").forward(d, g=g).cpu().numpy()
        assert O.max_abs_error(yb, ref) / np.abs(ref).max() <= REL_TOL[("bf16", m)]


@pytest.mark.parametrize("C", [1, 3, 6])
def test_small_c_layer(wb, C):
    """The whole-layer small-C kernel (C <= 8, VGG conv1.1): several filter
    chunks (K = 70 > 64, partial last chunk), partial 32-tile units along x,
    clipped edge tiles, every precision, against the fp64 direct conv and the
    oracle's fp32 Winograd."""
    import torch
    N, H, W, K = 2, 19, 75, 70
    cfg = wb.LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=1)
    dn = O.fill_uniform((N, C, H, W), 51 + C)
    gn = O.fill_uniform((K, C, 3, 3), 52 + C)
    ref = O.direct_forward(dn, gn, 1)
    for m in (2, 4):
        yo = O.winograd_forward(dn, gn, m, 1)
        for prec in ("fp32", "tf32", "bf16", "fp16"):
            plan = wb.WinogradPlan(cfg, m, prec)
            assert plan.info["fused_small_c"] == 1
            y = plan.forward(torch.from_numpy(dn).cuda(), g=torch.from_numpy(gn).cuda()).cpu().numpy()
            if prec == "fp32":
                assert O.max_abs_error(y, ref) < (5e-4 if m == 2 else 5e-3)
                assert np.abs(y - yo).max() <= 2e-5 * (1 + np.abs(yo).max())
            else:
                assert O.max_abs_error(y, ref) / np.abs(ref).max() <= REL_TOL[(prec, m)], prec
        if C <= 4 or m == 2:
            d64, g64 = dn.astype(np.float64), gn.astype(np.float64)
            y64 = _run(wb, d64, g64, 1, m)
            assert O.max_abs_error(y64, O.direct_forward(d64, g64, 1)) < 1e-12


@pytest.mark.parametrize("prec", ["bf16", "fp16"])
@pytest.mark.parametrize("m", [2, 4])
def test_bf16_staged_m_error_budget(wb, monkeypatch, m, prec):
    """The 16-bit GEMMs stage M in 16 bits (fp32 accumulation, one extra
    rounding of each accumulator: bf16, or fp16 of M * 2^-4).  Measured on
    B200 (tools/mbf16_error.py): bf16 +22-23% rms and +18-39% max-abs error
    over fp32-staged M; fp16 (emulated, tools/m16_emulation.py) +23% rms.
    Gates: within REL_TOL, rms error <= 1.35x the fp32-M plan's."""
    import torch
    monkeypatch.setenv("WINO_PATH", "staged")
    cfg = wb.LayerConfig(N=4, C=96, H=40, W=40, K=80, pad=1)  # enough tiles: no split-C
    dn = O.fill_uniform((4, 96, 40, 40), 61)
    gn = O.fill_uniform((80, 96, 3, 3), 62)
    d, g = torch.from_numpy(dn).cuda(), torch.from_numpy(gn).cuda()
    ref = O.direct_forward(dn, gn, 1)
    plan = wb.WinogradPlan(cfg, m, prec)
    assert plan.info["m_bytes_per_elem"] == 2
    e16 = plan.forward(d, g=g).cpu().numpy().astype(np.float64) - ref
    monkeypatch.setenv("WINO_M_FP32", "1")
    plan32 = wb.WinogradPlan(cfg, m, prec)
    assert plan32.info["m_bytes_per_elem"] == 4
    e32 = plan32.forward(d, g=g).cpu().numpy().astype(np.float64) - ref
    scale = np.abs(ref).max()
    assert np.abs(e16).max() / scale <= REL_TOL[(prec, m)]
    rms16, rms32 = np.sqrt((e16 ** 2).mean()), np.sqrt((e32 ** 2).mean())
    assert rms16 <= 1.35 * rms32, (rms16, rms32)


def test_presplit_filter_planes_bitwise(wb, monkeypatch):
    """Non-FX 3xTF32 plans with many tile blocks get U from the filter transform
    as hi / lo planes (no on-chip split of U in the GEMM); FX plans pass a
    one-plane U that the GEMM splits on chip.  Both feed the MMAs the same
    rna_tf32 hi and exact lo, so the outputs are bit-identical -- and within
    the fp32 gates of the oracle."""
    import torch
    monkeypatch.setenv("WINO_PATH", "staged")
    cfg = wb.LayerConfig(N=4, C=64, H=64, W=64, K=64, pad=1)
    dn = O.fill_uniform((4, 64, 64, 64), 71)
    gn = O.fill_uniform((64, 64, 3, 3), 72)
    d, g = torch.from_numpy(dn).cuda(), torch.from_numpy(gn).cuda()
    plan = wb.WinogradPlan(cfg, 2, "fp32")
    y_nonfx = plan.forward(d, g=g)
    y_fx = plan.forward(d, U=plan.filter_transform(g))
    torch.cuda.synchronize()
    assert torch.equal(y_nonfx, y_fx)
    y = y_nonfx.cpu().numpy()
    assert O.max_abs_error(y, O.direct_forward(dn, gn, 1)) < 5e-4
    yo = O.winograd_forward(dn, gn, 2, 1)
    assert np.abs(y - yo).max() <= 2e-5 * (1 + np.abs(yo).max())


@pytest.mark.parametrize("prec", ["bf16", "fp16"])
def test_tma_input_odd_channels_16bit(wb, prec):
    """TMA input transform with 16-bit operands and an odd channel count (a
    partial second block of 32 channels: zero-filled box channels past C must
    never be stored)."""
    import torch
    cfg = wb.LayerConfig(N=2, C=37, H=16, W=16, K=20, pad=1)
    dn = O.fill_uniform((2, 37, 16, 16), 81)
    gn = O.fill_uniform((20, 37, 3, 3), 82)
    d, g = torch.from_numpy(dn).cuda(), torch.from_numpy(gn).cuda()
    ref = O.direct_forward(dn, gn, 1)
    for m in (2, 4):
        y = wb.WinogradPlan(cfg, m, prec).forward(d, g=g).cpu().numpy()
        assert O.max_abs_error(y, ref) / np.abs(ref).max() <= REL_TOL[(prec, m)], (m, prec)


def test_cta_pair_gemm_variant_parity():
    """The cta_group::2 (CTA-pair) 3xTF32 GEMM variant, selected by
    WINO_GEMM_2SM=1 at first use in a fresh process, passes the fp32 gates
    (it is not the default: measured slower)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "gemm2sm_check.py")],
                         env={**os.environ, "WINO_GEMM_2SM": "1"}, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("N=")]
    assert len(lines) == 5 and all(l.endswith("OK") for l in lines), out.stdout


@pytest.mark.parametrize("pad", [0, 2, 3, 5])
def test_padding_variants(wb, pad):
    """Zero padding other than 1 (the TMA input box shifts by (-pad) mod 4, pad
    > 3 takes the generic staging kernel), F2 and F4, fp32 and bf16, W % 4 == 0
    and not."""
    for (H, W) in ((16, 20), (13, 10)):
        d = O.fill_uniform((2, 24, H, W), 90 + pad)
        g = O.fill_uniform((12, 24, 3, 3), 91 + pad)
        ref = O.direct_forward(d, g, pad)
        for m in (2, 4):
            y = _run(wb, d, g, pad, m)
            assert y.shape == ref.shape
            assert O.max_abs_error(y, ref) < (5e-4 if m == 2 else 5e-3), (pad, H, W, m)
            yb = _run(wb, d, g, pad, m, prec="bf16")
            assert O.max_abs_error(yb, ref) / np.abs(ref).max() <= REL_TOL[("bf16", m)]


@pytest.mark.parametrize("m", [2, 4])
@pytest.mark.parametrize("N,C,H,K", [
    (1, 40, 10, 136),   # P = 25 (F2) / 9 (F4): bn = 32 tiles, ragged K
    (1, 96, 15, 300),   # P = 64 / 16: bn = 64 / 32, K not a multiple of 128
    (2, 64, 19, 520),   # P = 200 / 50: bn = 128 (two tile blocks) / 64, ragged H
    (1, 512, 14, 512),  # conv5: split-C with the transposed GEMM
])
@pytest.mark.parametrize("vsplit", [True, False])
def test_transposed_gemm_k_gt_p(wb, monkeypatch, m, N, C, H, K, vsplit):
    """3xTF32 layers with more filters than tiles run the GEMM with the filters on
    the MMA's M side (TRN variant) and, by default, V pre-split into tf32 hi/lo
    planes by the input transform; both must meet the fp32 gates, and their
    error vs fp64 must not exceed the default-orientation GEMM's."""
    import torch
    if not vsplit:
        monkeypatch.setenv("WINO_NO_VSPLIT", "1")
    cfg = wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
    plan = wb.WinogradPlan(cfg, m, "fp32")
    th = (H + m - 1) // m
    assert plan.info["P"] == N * th * th < K
    d = O.fill_uniform((N, C, H, H), 41)
    g = O.fill_uniform((K, C, 3, 3), 42)
    dd, gg = torch.from_numpy(d).cuda(), torch.from_numpy(g).cuda()
    y = plan.forward(dd, g=gg).cpu().numpy()
    ref = O.direct_forward(d, g, 1)
    err = O.max_abs_error(y, ref)
    assert err < (5e-4 if m == 2 else 5e-3)
    # vs the reference's fp32 Winograd: tcgen05 truncates each accumulation, so
    # the gap grows with C (measured 2.7e-5 of max|y| at C = 512, F4); the
    # default-orientation GEMM is the yardstick for the error itself
    yo = O.winograd_forward(d, g, m, 1)
    assert np.abs(y - yo).max() <= (2e-5 if C <= 128 else 5e-5) * (1 + np.abs(yo).max())
    monkeypatch.setenv("WINO_NO_GEMM_TR", "1")
    y2 = wb.WinogradPlan(cfg, m, "fp32").forward(dd, g=gg).cpu().numpy()
    assert err <= 1.25 * O.max_abs_error(y2, ref) + 1e-6 * (1 + np.abs(ref).max())


# ---- winograd_grad_inputs (engine.py:257-275): the reference's TestGradInputs
# cases (test_engine.py:183-223) through the CUDA path, plus VGG-size layers.
def _grad_inputs_ref(dy, g, pad):
    """fp64 dL/dInput: correlation of dY with the flipped, (k,c)-swapped filters."""
    import torch
    flipped = torch.from_numpy(np.ascontiguousarray(
        g[:, :, ::-1, ::-1].transpose(1, 0, 2, 3))).double()
    return torch.nn.functional.conv2d(torch.from_numpy(dy).double(), flipped,
                                      padding=2 - pad).numpy()


def test_grad_inputs_zero_dy_exact(wb):
    cfg = wb.LayerConfig(N=1, C=2, H=6, W=6, K=3, pad=1)
    dy = wb.Tensor4.zeros((1, 3, 6, 6))
    g = wb.Tensor4.from_array(O.fill_uniform((3, 2, 3, 3), 1))
    for m in (2, 4):
        assert np.all(wb.winograd_grad_inputs(dy, g, cfg, wb.builtin(m, 3)).data == 0.0)


def test_grad_inputs_center_impulse_identity(wb):
    cfg = wb.LayerConfig(N=1, C=1, H=6, W=6, K=1, pad=1)
    g = np.zeros((1, 1, 3, 3))
    g[0, 0, 1, 1] = 1.0
    dy = O.fill_uniform((1, 1, 6, 6), 2).astype(np.float64)
    T = wb.Tensor4.from_array
    dd = wb.winograd_grad_inputs(T(dy, wb.Precision.FP64), T(g, wb.Precision.FP64), cfg,
                                 wb.builtin(2, 3)).data
    np.testing.assert_allclose(dd, dy, atol=1e-12)


@pytest.mark.parametrize("m", [2, 4])
def test_grad_inputs_matches_direct(wb, m):
    T = wb.Tensor4.from_array
    # fp64 (test_engine.py:201-207) and fp32 (test_engine.py:209-215) shapes
    cfg = wb.LayerConfig(N=1, C=1, H=8, W=8, K=1, pad=1)
    dy = O.fill_uniform((1, 1, 8, 8), 3).astype(np.float64)
    g = O.fill_uniform((1, 1, 3, 3), 4).astype(np.float64)
    dd = wb.winograd_grad_inputs(T(dy, wb.Precision.FP64), T(g, wb.Precision.FP64), cfg,
                                 wb.builtin(m, 3)).data
    assert O.max_abs_error(dd, _grad_inputs_ref(dy, g, 1)) < 1e-10
    cfg = wb.LayerConfig(N=2, C=3, H=9, W=7, K=4, pad=1)
    dy = O.fill_uniform((2, 4, 9, 7), 5)
    g = O.fill_uniform((4, 3, 3, 3), 6)
    dd = wb.winograd_grad_inputs(T(dy), T(g), cfg, wb.builtin(m, 3)).data
    assert O.max_abs_error(dd, _grad_inputs_ref(dy, g, 1)) < 1e-3


def test_grad_inputs_pad_too_large(wb):
    cfg = wb.LayerConfig(N=1, C=1, H=6, W=6, K=1, pad=3)
    dy = wb.Tensor4.from_array(O.fill_uniform((1, 1, cfg.out_h, cfg.out_w), 7))
    g = wb.Tensor4.from_array(O.fill_uniform((1, 1, 3, 3), 8))
    with pytest.raises(ValueError):
        wb.winograd_grad_inputs(dy, g, cfg, wb.builtin(2, 3))


@pytest.mark.parametrize("m", [2, 4])
@pytest.mark.parametrize("C,H,K,pad", [(256, 56, 256, 1), (512, 14, 512, 1), (64, 30, 96, 0),
                                       (128, 28, 64, 2)])
def test_grad_inputs_vgg_size(wb, m, C, H, K, pad):
    """VGG-size layers (the deep and small-C-out shapes, pad 0 / 1 / 2) against the
    fp64 gradient, at the fp32 forward gates."""
    T = wb.Tensor4.from_array
    cfg = wb.LayerConfig(N=1, C=C, H=H, W=H, K=K, pad=pad)
    dy = O.fill_uniform((1, K, cfg.out_h, cfg.out_w), 11)
    g = O.fill_uniform((K, C, 3, 3), 12)
    dd = wb.winograd_grad_inputs(T(dy), T(g), cfg, wb.builtin(m, 3)).data
    assert dd.shape == (1, C, H, H)
    assert O.max_abs_error(dd, _grad_inputs_ref(dy, g, pad)) < (5e-4 if m == 2 else 5e-3)


@pytest.mark.parametrize("m", [2, 4])
@pytest.mark.parametrize("N,C,H,K", [(1, 512, 14, 512), (1, 96, 15, 300), (2, 40, 10, 136)])
@pytest.mark.parametrize("prec", ["tf32", "bf16", "fp16"])
def test_single_pass_transposed_gemm(wb, monkeypatch, m, N, C, H, K, prec):
    """tf32 / bf16 / fp16 plans with K > P <= 64 put the filters on the MMA's
    128-row side (the 3xTF32 TRN orientation, fp32 M): same gates as the default
    orientation, which WINO_NO_GEMM_TR16=1 restores."""
    import torch
    monkeypatch.setenv("WINO_PATH", "staged")
    cfg = wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
    plan = wb.WinogradPlan(cfg, m, prec)
    P = plan.info["P"]
    if P > 64:
        pytest.skip(f"P = {P} > 64: default orientation")
    assert plan.info["gemm_bn"] in (32, 64) and plan.info["m_bytes_per_elem"] == 4
    d = O.fill_uniform((N, C, H, H), 71)
    g = O.fill_uniform((K, C, 3, 3), 72)
    dd, gg = torch.from_numpy(d).cuda(), torch.from_numpy(g).cuda()
    y = plan.forward(dd, g=gg).cpu().numpy()
    ref = O.direct_forward(d, g, 1)
    scale = np.abs(ref).max()
    err = O.max_abs_error(y, ref) / scale
    assert err <= REL_TOL[(prec, m)], err
    monkeypatch.setenv("WINO_NO_GEMM_TR16", "1")
    y0 = wb.WinogradPlan(cfg, m, prec).forward(dd, g=gg).cpu().numpy()
    err0 = O.max_abs_error(y0, ref) / scale
    assert err <= 1.5 * err0 + 1e-6, (err, err0)
