"""Pin the CPU oracle to the reference: every check compares oracle/ against
fixtures produced by the real reference (tests/golden/make_golden.py)."""
import numpy as np
import pytest

from oracle import winograd_oracle as O


@pytest.mark.parametrize("seed", [0, 1, 7, 12345, 2**63 + 5, 2**64 - 1])
def test_splitmix64_stream(golden, seed):
    assert np.array_equal(O.splitmix64_unit(257, seed), golden[f"sm64_{seed}"])


def test_fill_uniform(golden):
    assert np.array_equal(O.fill_uniform((2, 3, 5, 7), 3), golden["fill_f32_s3"])
    assert np.array_equal(O.fill_uniform((1, 2, 3, 4), 4, dtype=np.float64), golden["fill_f64_s4"])
    assert np.array_equal(O.fill_uniform((1, 1, 4, 64), 9, -0.5, 2.0), golden["fill_f32_lohi"])
    q = O.quantize_fp16(O.fill_uniform((1, 2, 8, 8), 11))
    assert np.array_equal(q, golden["fp16_q"])


@pytest.mark.parametrize("mr", [(2, 3), (4, 3), (3, 2)])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_lowered_matrices(golden, mr, dt):
    m, r = mr
    BT, G, AT = O.lowered(m, r, dt)
    tag = np.dtype(dt).name
    assert np.array_equal(BT, golden[f"BT_{m}{r}_{tag}"])
    assert np.array_equal(G, golden[f"G_{m}{r}_{tag}"])
    assert np.array_equal(AT, golden[f"AT_{m}{r}_{tag}"])


def test_unknown_builtin():
    with pytest.raises(KeyError):
        O.exact_matrices(3, 3)


def test_tile_grid(golden):
    for row in golden["tile_grid"]:
        N, C, H, W, K, pad, m, th, tw, P, tc, mul, b, n, ty, tx, oy, ox = (int(v) for v in row)
        oh, ow = O.out_dims(H, W, 3, 3, pad)
        assert O.tile_grid(N, oh, ow, m) == (th, tw, P)
        assert P == tc and mul == P * C * K * (m + 2) ** 2
        assert O.tile_index(b, N, th, tw) == (n, ty, tx)
        assert (m * ty - pad, m * tx - pad) == (oy, ox)
    with pytest.raises(IndexError):
        O.tile_index(4, 1, 2, 2)


@pytest.mark.parametrize("i", range(10))
def test_whole_layer_bit_exact(golden, i):
    """Oracle winograd_forward == reference winograd_forward, bit for bit,
    fp32 and fp64, both algorithms; direct_forward fp64 bit-exact too."""
    N, C, H, W, K, pad = (int(v) for v in golden[f"case{i}_shape"])
    d = O.fill_uniform((N, C, H, W), 100 + 2 * i)
    g = O.fill_uniform((K, C, 3, 3), 101 + 2 * i)
    assert np.array_equal(O.direct_forward(d, g, pad), golden[f"case{i}_direct64"])
    for m in (2, 4):
        assert np.array_equal(O.winograd_forward(d, g, m, pad), golden[f"case{i}_f{m}_fp32"])
        assert np.array_equal(O.winograd_forward(d.astype(np.float64), g.astype(np.float64), m,
                                                 pad), golden[f"case{i}_f{m}_fp64"])
        if f"case{i}_f{m}_U" in golden:
            assert np.array_equal(O.filter_transform(g, m), golden[f"case{i}_f{m}_U"])
        # FX variant (precomputed U) is bitwise transparent (engine.py:117-160)
        U = O.filter_transform(g, m)
        assert np.array_equal(O.winograd_forward(d, g, m, pad, U=U), golden[f"case{i}_f{m}_fp32"])
    dq, gq = O.quantize_fp16(d), O.quantize_fp16(g)
    assert np.array_equal(O.winograd_forward(dq, gq, 4, pad), golden[f"case{i}_f4_fp16sim"])


def test_config1_sample(golden):
    d = O.fill_uniform((1, 64, 56, 56), 0)
    g = O.fill_uniform((64, 64, 3, 3), 1)
    for m in (2, 4):
        y = O.winograd_forward(d, g, m, 1)
        assert np.array_equal(y.reshape(-1)[::37], golden[f"cfg1_f{m}_sample"])


def test_numpy_gemm_matches_numba_order():
    u = O.fill_uniform((3, 5, 7), 1)
    v = O.fill_uniform((3, 7, 9), 2)
    assert np.array_equal(O._bgemm_numpy(u, v), O.batched_matmul(u, v))


def test_vgg_e_gflops():
    total = sum(O.gflops_direct(1, C, H, H, K, 1, depth=dep) for _, C, H, K, dep in O.VGG_E)
    assert round(total, 2) == 39.02  # PAPER.md:485-509, test_suites.py:17-18
