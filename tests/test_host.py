"""Host-side logic of the drop-in (no GPU needed): interface types, tile
grid, planner, validation errors -- mirroring the reference's unit tests
(test_engine.py:17-71,128-139; test_tensors.py; test_suites.py)."""
import re

import numpy as np
import pytest

import paper_1509_09308_b200 as wb
from paper_1509_09308_b200 import engine, sharding


def rand(shape, seed, prec=wb.Precision.FP32):
    return wb.fill_uniform(wb.Tensor4.zeros(shape, precision=prec), seed, -1.0, 1.0)


def test_fill_uniform_matches_reference(golden):
    assert np.array_equal(rand((2, 3, 5, 7), 3).data, golden["fill_f32_s3"])
    assert np.array_equal(rand((1, 2, 3, 4), 4, wb.Precision.FP64).data, golden["fill_f64_s4"])
    t = wb.fill_uniform(wb.Tensor4.zeros((1, 1, 4, 64)), 9, -0.5, 2.0)
    assert np.array_equal(t.data, golden["fill_f32_lohi"])
    assert np.array_equal(wb.quantize_fp16(rand((1, 2, 8, 8), 11)).data, golden["fp16_q"])


def test_tensor4_contract():
    t = rand((1, 2, 3, 4), 1)
    assert not t.data.flags.writeable
    with pytest.raises(IndexError):
        t[0, 2, 0, 0]
    with pytest.raises(ValueError):
        wb.Tensor4(np.zeros((2, 2)), wb.Precision.FP32)
    with pytest.raises(ValueError):
        wb.fill_uniform(t, 0, 1.0, 1.0)
    with pytest.raises(OverflowError):
        wb.quantize_fp16(wb.Tensor4.from_array(np.full((1, 1, 1, 1), 1e6)))


@pytest.mark.parametrize("mr", [(2, 3), (4, 3)])
def test_builtin_matrices_match_reference(golden, mr):
    m, r = mr
    alg = wb.builtin(m, r)
    for dt in (np.float32, np.float64):
        BT, G, AT = alg.lowered(dt)
        tag = np.dtype(dt).name
        assert np.array_equal(BT, golden[f"BT_{m}{r}_{tag}"])
        assert np.array_equal(G, golden[f"G_{m}{r}_{tag}"])
        assert np.array_equal(AT, golden[f"AT_{m}{r}_{tag}"])
    assert alg.alpha == m + 2


def test_cuda_constants_match_reference(golden):
    """The kernels' compiled-in matrices (csrc/winograd_mats.cuh) equal the
    reference's lowered matrices entry by entry."""
    import os
    src = open(os.path.join(os.path.dirname(wb.__file__), "csrc", "winograd_mats.cuh")).read()
    for m, r, n in ((2, 3, 4), (4, 3, 6)):
        body = src[src.index(f"struct Alg<{m}>"):]
        for name, rows in (("BT", n), ("G", n), ("AT", m)):
            blk = body[body.index(f"double {name}("):]
            blk = blk[blk.index("= {") + 2: blk.index("};")]
            vals = [eval(v) for v in re.findall(r"-?[\d.]+(?:\s*/\s*\d+)?", blk)]
            ref = golden[f"{name}_{m}{r}_float64"]
            assert np.array_equal(np.array(vals).reshape(ref.shape), ref), (m, name)
            assert np.array_equal(np.array(vals, np.float32).reshape(ref.shape),
                                  golden[f"{name}_{m}{r}_float32"])


def test_unknown_builtin():
    with pytest.raises(KeyError):
        wb.builtin(3, 3)


def test_tile_grid_matches_reference(golden):
    for row in golden["tile_grid"]:
        N, C, H, W, K, pad, m, th, tw, P, tc, mul, b, n, ty, tx, oy, ox = (int(v) for v in row)
        cfg = wb.LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=pad)
        grid = wb.TileGrid.for_layer(cfg, m, 3)
        assert (grid.tiles_h, grid.tiles_w, grid.P) == (th, tw, P)
        assert wb.tile_count(cfg, m) == tc
        assert wb.multiply_stage_flops(cfg, m) == mul
        assert grid.index(b) == (n, ty, tx) and grid.origin(b) == (oy, ox)
    with pytest.raises(IndexError):
        grid.index(grid.P)


def test_reference_counts():
    # test_engine.py:47-58
    assert wb.tile_count(wb.LayerConfig(N=1, C=1, H=224, W=224, K=1, pad=1), 2) == 12544
    assert wb.tile_count(wb.LayerConfig(N=1, C=1, H=14, W=14, K=1, pad=1), 4) == 16
    cfg = wb.LayerConfig(N=2, C=3, H=9, W=7, K=5, pad=1)
    assert wb.multiply_stage_flops(cfg, 1) == 2 * cfg.out_h * cfg.out_w * 3 * 5 * 9


def test_layer_config_validation():
    with pytest.raises(ValueError):
        wb.LayerConfig(N=0, C=1, H=4, W=4, K=1)
    with pytest.raises(ValueError):
        wb.LayerConfig(N=1, C=1, H=4, W=4, K=1, pad=-1)
    with pytest.raises(ValueError):
        wb.LayerConfig(N=1, C=1, H=2, W=2, K=1, pad=0)


def test_forward_validation_errors_before_gpu():
    """engine.py:211-218 error paths raise ValueError without touching the GPU."""
    cfg = wb.LayerConfig(N=1, C=1, H=6, W=6, K=1, pad=1)
    d32 = rand((1, 1, 6, 6), 1)
    g64 = rand((1, 1, 3, 3), 2, wb.Precision.FP64)
    with pytest.raises(ValueError):
        wb.winograd_forward(d32, g64, cfg, wb.builtin(2, 3))
    with pytest.raises(ValueError):
        wb.winograd_forward(rand((1, 2, 6, 6), 1), rand((1, 1, 3, 3), 2), cfg)
    cfg2 = wb.LayerConfig(N=1, C=1, H=6, W=6, K=1, R=2, S=2, pad=0)
    with pytest.raises(ValueError):
        wb.winograd_forward(rand((1, 1, 6, 6), 1), rand((1, 1, 2, 2), 2), cfg2, wb.builtin(2, 3))
    with pytest.raises(ValueError):
        wb.run_layer("f8x8", d32, rand((1, 1, 3, 3), 2), cfg)


def test_plan_info_and_planner():
    cfg = wb.LayerConfig(N=1, C=64, H=56, W=56, K=64, pad=1)
    p = wb.WinogradPlan(cfg, 2, "fp32")
    i = p.info
    assert (i["tiles_h"], i["tiles_w"], i["P"], i["alpha"]) == (28, 28, 784, 4)
    assert i["multiplies"] == wb.multiply_stage_flops(cfg, 2)
    # 3xTF32 stores one fp32 plane in HBM (hi/lo split on chip)
    assert i["op_splits"] == 1 and i["op_bytes"] == 4 and i["num_chunks"] == 1
    # the chunk planner respects the workspace budget with whole tile rows
    big = wb.LayerConfig(N=64, C=64, H=224, W=224, K=64, pad=1)
    for m, prec in ((4, "bf16"), (2, "fp32")):
        q = wb.WinogradPlan(big, m, prec, workspace_limit=32 << 20)
        j = q.info
        per_tile = j["op_splits"] * j["op_bytes"] * (m + 2) ** 2 * j["c_pad"] + (m + 2) ** 2 * 64 * 4
        assert j["chunk_tiles"] % j["tiles_w"] == 0
        assert j["chunk_tiles"] * per_tile <= 32 << 20
        assert j["num_chunks"] * j["rows_per_chunk"] >= 64 * j["tiles_h"]
        assert j["launches_per_forward"] == 3 * j["num_chunks"]


def test_plan_errors_map_to_reference_exceptions():
    with pytest.raises(ValueError):
        wb.WinogradPlan(wb.LayerConfig(N=1, C=1, H=6, W=6, K=1, pad=1), 3, "fp32")
    with pytest.raises(ValueError):
        wb.WinogradPlan(wb.LayerConfig(N=1, C=1, H=6, W=6, K=1, pad=1), 2, "int8")
    with pytest.raises(ValueError):
        wb.WinogradPlan(wb.LayerConfig(N=1, C=1, H=6, W=6, K=1, R=5, S=5, pad=2), 2, "fp32")


def test_bench_algo_names_match_reference():
    """cmd_bench accepts the reference's full BENCH_ALGOS (commands.py:26) and
    rejects anything else with the reference's ValueError."""
    assert wb.BENCH_ALGOS == ("direct", "direct-fp32", "f2x2", "f4x4", "f2x2-fx", "f4x4-fx",
                              "fft")
    with pytest.raises(ValueError, match="unknown algorithm"):
        wb.cmd_bench(algo="f3x3")
    with pytest.raises(ValueError, match="repeats"):
        wb.cmd_bench(algo="direct", repeats=0)


def test_parse_algo():
    assert wb.parse_algo("f2x2") == (2, False, None)
    assert wb.parse_algo("f4x4-fx:bf16") == (4, True, "bf16")
    with pytest.raises(ValueError):
        wb.parse_algo("fft")
    with pytest.raises(ValueError):
        wb.parse_algo("f4x4:int4")


def test_suites():
    s = wb.vgg_e()
    assert len(s.entries) == 9 and round(s.total_gflops_direct(), 2) == 39.02
    assert sum(e.cfg.depth for e in s.entries) == 16
    sc = s.scaled(0.05)
    assert all(e.cfg.H >= 3 for e in sc.entries)
    assert all(e.cfg.N == 8 for e in s.with_batch(8).entries)
    assert wb.get_suite("vgg-e-accuracy").labels() == ("conv1.2", "conv2.2", "conv3.2",
                                                        "conv4.2", "conv5")


def test_counter():
    c = wb.OpCounter()
    c.add("mul", 3)
    c.add("mul", 4)
    assert c["mul"] == 7 and c.get("cmul") == 0
    with pytest.raises(ValueError):
        c.add("mul", -1)


@pytest.mark.parametrize("N,world", [(64, 8), (64, 3), (5, 8), (1, 1), (7, 2)])
def test_shard_bounds_partition(N, world):
    spans = [sharding.shard_bounds(N, world, r) for r in range(world)]
    assert sum(c for _, c in spans) == N
    pos = 0
    for s, c in spans:
        assert s == pos
        pos += c
    assert max(c for _, c in spans) - min(c for _, c in spans) <= 1

    # the C ABI's wino_shard_bounds is the same split (host-only call)
    assert [sharding.shard_bounds_native(N, world, r) for r in range(world)] == spans


def test_shard_abi_errors_and_workspace():
    import ctypes
    from paper_1509_09308_b200 import _lib
    with pytest.raises(ValueError):
        sharding.shard_bounds_native(8, 0, 0)
    with pytest.raises(ValueError):
        sharding.shard_bounds_native(8, 2, 2)
    cfg = wb.LayerConfig(N=5, C=64, H=28, W=28, K=64, pad=1)
    plan = engine.WinogradPlan(cfg, 4, "bf16")
    b = ctypes.c_size_t()
    for s, cnt in enumerate((2, 2, 1)):
        sub = engine.WinogradPlan(cfg.with_batch(cnt), 4, "bf16")
        for with_g, key in ((1, "workspace_bytes"), (0, "staging_bytes")):
            assert _lib.lib.wino_shard_workspace(plan._h, 3, s, with_g, ctypes.byref(b)) == 0
            assert b.value == sub.info[key]
    # a shard without images needs nothing
    assert _lib.lib.wino_shard_workspace(plan._h, 8, 7, 1, ctypes.byref(b)) == 0 and b.value == 0
    assert _lib.lib.wino_forward_sharded(plan._h, 0, None, None, None, None, None, None, None,
                                         None) == _lib.WINO_EINVAL

def test_filter_cache_key_semantics():
    g = rand((2, 3, 3, 3), 1)
    alg = wb.builtin(4, 3)
    k1 = engine.FilterCache._key(g, alg, "fp32")
    assert k1 == engine.FilterCache._key(rand((2, 3, 3, 3), 1), alg, "fp32")
    assert k1 != engine.FilterCache._key(rand((2, 3, 3, 3), 2), alg, "fp32")
    assert k1 != engine.FilterCache._key(g, alg, "bf16")
    assert k1 != engine.FilterCache._key(g, wb.builtin(2, 3), "fp32")


def test_cli_bench_usage_errors():
    """The bench CLI maps domain errors to exit code 1 (reference cli.py:150-159)."""
    from paper_1509_09308_b200.__main__ import main
    assert main(["bench", "--algo", "fft2"]) == 1
    assert main(["bench", "--algo", "f4x4:int8"]) == 1
    assert main(["bench", "--batch", "0"]) == 1


def test_report_text_and_csv():
    from paper_1509_09308_b200.commands import Report
    r = Report(columns=("layer", "algo", "batch", "msec", "effective_gflops"), seed=3)
    r.add("conv1.1", "f4x4", 1, 0.5, 123.25)
    r.add("conv1.2", "f4x4", 1, None, None)
    assert r.to_csv().splitlines()[0] == "# seed=3"
    assert "conv1.1,f4x4,1,0.5,123.25" in r.to_csv()
    txt = r.to_text()
    assert "conv1.1" in txt and "123.2" in txt and "-" in txt.splitlines()[-1]


def test_planner_decisions_vgg():
    """The C planner's choices on VGG-E layers (plan creation needs no GPU):
    split-C from the waves x k-steps cost model, bf16-staged M, two chunk
    buffers for multi-chunk staged plans, pre-split U workspace for large P."""
    import paper_1509_09308_b200 as wb

    def info(C, H, K, m, prec, N):
        return wb.WinogradPlan(wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1), m, prec).info

    conv5 = info(512, 14, 512, 2, "fp32", 1)      # 1 tile block x 4 x 16 = 64 units
    assert conv5["gemm_splits"] == 2 and conv5["m_bytes_per_elem"] == 4
    conv42 = info(512, 28, 512, 2, "fp32", 1)     # 128 units: one wave without a split
    assert conv42["gemm_splits"] == 1
    conv32 = info(256, 56, 256, 4, "bf16", 64)
    assert conv32["m_bytes_per_elem"] == 2 and conv32["num_chunks"] > 1
    # fp16 stages M in fp16 (x 2^-4) too, small single F(4x4) chunks included
    # (WINO_OUT_TMA_MIN=0); the transposed GEMM (K > P <= 64) keeps fp32 M
    assert info(256, 56, 256, 4, "fp16", 64)["m_bytes_per_elem"] == 2
    assert info(256, 56, 256, 4, "fp16", 1)["m_bytes_per_elem"] == 2
    assert info(512, 14, 512, 4, "fp16", 1)["m_bytes_per_elem"] == 4
    assert info(64, 224, 64, 4, "fp16", 1)["m_bytes_per_elem"] == 2
    conv12 = info(64, 224, 64, 2, "fp32", 64)
    assert conv12["num_chunks"] > 1 and conv12["m_bytes_per_elem"] == 4
    # large-P 3xTF32: workspace holds U as hi/lo planes (2 x u_bytes) + two V/M chunk sets
    assert conv12["workspace_bytes"] >= 2 * conv12["u_bytes"]


def test_cli_accuracy_usage_errors():
    from paper_1509_09308_b200.__main__ import main
    assert main(["accuracy", "--algos", "fft8"]) == 1
    assert main(["accuracy", "--algos", "f2x2", "--suite", "no-such-suite"]) == 1


def test_vgg_e_network_layers():
    """network E's 16 conv layers in order, with a pool closing each block
    (PAPER.md:549-563): 224 -> 112 -> 56 -> 28 -> 14 -> 7."""
    from paper_1509_09308_b200.network import vgg_e_layers
    layers = vgg_e_layers()
    assert len(layers) == 16
    assert [l[0] for l in layers][:3] == ["conv1.1", "conv1.2", "conv2.1"]
    chans = [(C, K) for (_, C, _, K, _) in layers]
    assert all(chans[i][1] == chans[i + 1][0] for i in range(15))  # K_i == C_{i+1}
    pools = [i for i, l in enumerate(layers) if l[4]]
    assert pools == [1, 3, 7, 11, 15]
    sizes = [H for (_, _, H, _, _) in layers]
    for i in pools[:-1]:
        assert sizes[i + 1] == sizes[i] // 2


def test_forward_act_shapes_and_validation():
    """act="relu_pool" halves the output plane; unknown activations are rejected
    before any launch (plan creation needs no GPU)."""
    import paper_1509_09308_b200 as wb
    plan = wb.WinogradPlan(wb.LayerConfig(N=2, C=16, H=28, W=28, K=8, pad=1), 4, "fp32")
    assert plan.act_shape(None) == plan.out_shape == (2, 8, 28, 28)
    assert plan.act_shape("relu") == (2, 8, 28, 28)
    assert plan.act_shape("relu_pool") == (2, 8, 14, 14)
    with pytest.raises(ValueError):
        plan.forward(None, act="gelu")
