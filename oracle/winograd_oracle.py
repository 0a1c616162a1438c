"""CPU oracle for the Winograd forward path -- TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy (+ optional numba) restatement of the
reference algorithm in ``winoconv`` (``/root/reference/pkg/src/winoconv``).
It exists so the CUDA path can be checked against the reference's own
arithmetic on identical inputs.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it;
the product package (``paper_1509_09308_b200``) never does.

Parity is PINNED: ``tests/golden/make_golden.py`` imports the real reference
in the build container and records its outputs (SplitMix64 streams, lowered
transform matrices, tile grids, whole-layer ``winograd_forward`` and
``direct_forward`` results); ``tests/test_oracle_golden.py`` checks every
function below against those fixtures.

Each function cites the reference file:line it restates.
"""
from __future__ import annotations

import os
from fractions import Fraction
from typing import Dict, Tuple

import numpy as np

# ---------------------------------------------------------------------------
# SplitMix64 counter-based uniform fill  (tensors.py:122-153)
# ---------------------------------------------------------------------------
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def splitmix64_unit(count: int, seed: int) -> np.ndarray:
    """Stream element i -> finalizer(seed + (i+1)*gamma), top 53 bits / 2**53.

    Restates ``_splitmix64_unit_doubles`` (tensors.py:122-135).
    """
    with np.errstate(over="ignore"):
        state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + \
            np.arange(1, count + 1, dtype=np.uint64) * _GAMMA
        state = (state ^ (state >> np.uint64(30))) * _MIX1
        state = (state ^ (state >> np.uint64(27))) * _MIX2
        state = state ^ (state >> np.uint64(31))
    return (state >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def fill_uniform(shape, seed: int, lo: float = -1.0, hi: float = 1.0,
                 dtype=np.float32) -> np.ndarray:
    """Uniform [lo, hi) array, bit-identical to ``fill_uniform`` (tensors.py:138-153)."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) if len(shape) else 1
    vals = (lo + splitmix64_unit(n, seed) * (hi - lo)).astype(dt)
    ceiling = np.nextafter(dt.type(hi), dt.type(lo))
    vals[vals.astype(np.float64) >= float(hi)] = ceiling
    return vals.reshape(shape)


def quantize_fp16(x: np.ndarray) -> np.ndarray:
    """RNE snap to binary16, stored at fp32 (tensors.py:156-169)."""
    return x.astype(np.float16).astype(np.float32)


def max_abs_error(a: np.ndarray, b: np.ndarray) -> float:
    """max |a-b| at fp64 (tensors.py:172-179)."""
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a.astype(np.float64) - b.astype(np.float64))))


# ---------------------------------------------------------------------------
# Builtin F(m, r) transform matrices  (winograd.py:151-215)
# ---------------------------------------------------------------------------
def _fr(rows):
    return [[Fraction(v) for v in row] for row in rows]


_H = Fraction(1, 2)
_MATS: Dict[Tuple[int, int], Tuple[list, list, list]] = {
    # (BT, G, AT) for F(2,3)  (winograd.py:151-168)
    (2, 3): (
        _fr([[1, 0, -1, 0], [0, 1, 1, 0], [0, -1, 1, 0], [0, 1, 0, -1]]),
        _fr([[1, 0, 0], [_H, _H, _H], [_H, -_H, _H], [0, 0, 1]]),
        _fr([[1, 1, 1, 0], [0, 1, -1, -1]]),
    ),
    # F(3,2)  (winograd.py:171-189) -- used only by the weight-gradient path
    (3, 2): (
        _fr([[1, 0, -1, 0], [0, 1, 1, 0], [0, -1, 1, 0], [0, -1, 0, 1]]),
        _fr([[1, 0], [_H, _H], [_H, -_H], [0, 1]]),
        _fr([[1, 1, 1, 0], [0, 1, -1, 0], [0, 1, 1, 1]]),
    ),
    # F(4,3)  (winograd.py:192-215)
    (4, 3): (
        _fr([[4, 0, -5, 0, 1, 0], [0, -4, -4, 1, 1, 0], [0, 4, -4, -1, 1, 0],
             [0, -2, -1, 2, 1, 0], [0, 2, -1, -2, 1, 0], [0, 4, 0, -5, 0, 1]]),
        _fr([[Fraction(1, 4), 0, 0],
             [Fraction(-1, 6), Fraction(-1, 6), Fraction(-1, 6)],
             [Fraction(-1, 6), Fraction(1, 6), Fraction(-1, 6)],
             [Fraction(1, 24), Fraction(1, 12), Fraction(1, 6)],
             [Fraction(1, 24), Fraction(-1, 12), Fraction(1, 6)],
             [0, 0, 1]]),
        _fr([[1, 1, 1, 1, 1, 0], [0, 1, -1, 2, -2, 0],
             [0, 1, 1, 4, 4, 0], [0, 1, -1, 8, -8, 1]]),
    ),
}


def exact_matrices(m: int, r: int):
    """Exact rational (BT, G, AT); KeyError for unknown sizes (winograd.py:225-232)."""
    try:
        return _MATS[(m, r)]
    except KeyError:
        raise KeyError(f"no builtin algorithm for F({m},{r})") from None


def lowered(m: int, r: int, dtype=np.float32):
    """Round each rational entry once to ``dtype`` (engine.py:98-101, rational.py:135-141)."""
    def low(rows):
        return np.array([[float(v) for v in row] for row in rows], dtype=dtype)
    bt, g, at = exact_matrices(m, r)
    return low(bt), low(g), low(at)


# ---------------------------------------------------------------------------
# Tile grid  (engine.py:40-95)
# ---------------------------------------------------------------------------
def out_dims(H: int, W: int, R: int, S: int, pad: int) -> Tuple[int, int]:
    """(direct.py:57-63)"""
    return H + 2 * pad - R + 1, W + 2 * pad - S + 1


def tile_grid(N: int, out_h: int, out_w: int, m: int) -> Tuple[int, int, int]:
    """(tiles_h, tiles_w, P) with ceil division (engine.py:57-69)."""
    th = -(-out_h // m)
    tw = -(-out_w // m)
    return th, tw, N * th * tw


def tile_index(b: int, N: int, th: int, tw: int) -> Tuple[int, int, int]:
    """Row-major tile id -> (n, ty, tx) (engine.py:71-76)."""
    if not 0 <= b < N * th * tw:
        raise IndexError(b)
    n, rest = divmod(b, th * tw)
    ty, tx = divmod(rest, tw)
    return n, ty, tx


# ---------------------------------------------------------------------------
# Deterministic batched GEMM  (kernels.py:31-65)
# ---------------------------------------------------------------------------
def _bgemm_numpy(u: np.ndarray, v: np.ndarray) -> np.ndarray:
    # c-ascending accumulation, one output row at a time (same order as
    # kernels.py:43-47), vectorised over p.
    B, K, C = u.shape
    out = np.zeros((B, K, v.shape[2]), dtype=u.dtype)
    for c in range(C):
        out += u[:, :, c, None] * v[:, None, c, :]
    return out


_bgemm = None
try:  # numba makes the oracle usable as a CPU baseline at VGG sizes
    if os.environ.get("WINO_ORACLE_NO_NUMBA") != "1":
        import numba as _nb

        @_nb.njit(parallel=True, cache=False)
        def _bgemm_nb(u, v, out):  # pragma: no cover - compiled
            nb, nk, nc = u.shape
            np_ = v.shape[2]
            for row in _nb.prange(nb * nk):
                b = row // nk
                k = row - b * nk
                acc = out[b, k]
                for p in range(np_):
                    acc[p] = 0.0
                for c in range(nc):
                    s = u[b, k, c]
                    src = v[b, c]
                    for p in range(np_):
                        acc[p] += s * src[p]

        _bgemm = _bgemm_nb
except Exception:  # pragma: no cover
    _bgemm = None


def batched_matmul(u: np.ndarray, v: np.ndarray) -> np.ndarray:
    """out[b] = u[b] @ v[b] accumulating over c in ascending order (kernels.py:50-65)."""
    u = np.ascontiguousarray(u)
    v = np.ascontiguousarray(v)
    if _bgemm is None:
        return _bgemm_numpy(u, v)
    out = np.empty((u.shape[0], u.shape[1], v.shape[2]), dtype=u.dtype)
    _bgemm(u, v, out)
    return out


def set_threads(n: int) -> int:
    """Cap numba threads (kernels.py:23-28); returns the count in use."""
    try:
        import numba
        n = max(1, min(int(n), numba.config.NUMBA_NUM_THREADS))
        numba.set_num_threads(n)
        return n
    except Exception:
        return 1


def threads_in_use() -> int:
    try:
        import numba
        return int(numba.get_num_threads()) if _bgemm is not None else 1
    except Exception:
        return 1


# ---------------------------------------------------------------------------
# Transforms and the whole-layer forward  (engine.py:104-254)
# ---------------------------------------------------------------------------
def filter_transform(g: np.ndarray, m: int) -> np.ndarray:
    """U[xi*alpha+nu, k, c] = (G g_kc G^T)[xi, nu]  (engine.py:104-114)."""
    K, C, R, S = g.shape
    _, G, _ = lowered(m, R, g.dtype)
    a = G.shape[0]
    rows = np.einsum("xr,kcrs->xkcs", G, g)
    full = np.einsum("ys,xkcs->xykc", G, rows)
    return np.ascontiguousarray(full.reshape(a * a, K, C))


def gather_tiles(d: np.ndarray, th: int, tw: int, step: int, span: int,
                 pad: int) -> np.ndarray:
    """Zero-filled overlapping span x span patches, (N, th, tw, C, span, span)
    (engine.py:170-191).  Out-of-range pixels stay 0: padding is virtual."""
    N, C, H, W = d.shape
    out = np.zeros((N, th, tw, C, span, span), dtype=d.dtype)
    for ty in range(th):
        y0 = step * ty - pad
        ya, yb = max(y0, 0), min(y0 + span, H)
        if ya >= yb:
            continue
        for tx in range(tw):
            x0 = step * tx - pad
            xa, xb = max(x0, 0), min(x0 + span, W)
            if xa >= xb:
                continue
            out[:, ty, tx, :, ya - y0:yb - y0, xa - x0:xb - x0] = d[:, :, ya:yb, xa:xb]
    return out


def input_transform(d: np.ndarray, m: int, pad: int, r: int = 3):
    """V (alpha^2, C, P) from data (engine.py:232-237); returns (V, th, tw)."""
    N, C, H, W = d.shape
    BT, _, _ = lowered(m, r, d.dtype)
    a = BT.shape[0]
    oh, ow = out_dims(H, W, r, r, pad)
    th, tw, P = tile_grid(N, oh, ow, m)
    tiles = gather_tiles(d, th, tw, m, a, pad).reshape(P, C, a, a)
    t = np.einsum("xu,pcuv->xpcv", BT, tiles)
    V = np.einsum("yv,xpcv->xycp", BT, t)
    return np.ascontiguousarray(V.reshape(a * a, C, P)), th, tw


def output_transform(M: np.ndarray, m: int, K: int, N: int, th: int, tw: int,
                     out_h: int, out_w: int, r: int = 3) -> np.ndarray:
    """Y = A^T M A per tile, clipped write-back (engine.py:241-254)."""
    _, _, AT = lowered(m, r, M.dtype)
    a = AT.shape[1]
    P = N * th * tw
    M4 = M.reshape(a, a, K, P)
    t2 = np.einsum("mx,xykp->mykp", AT, M4)
    Yt = np.einsum("ny,mykp->mnkp", AT, t2).reshape(m, m, K, N, th, tw)
    out = np.zeros((N, K, out_h, out_w), dtype=M.dtype)
    for ty in range(th):
        vr = min(m, out_h - m * ty)
        for tx in range(tw):
            vc = min(m, out_w - m * tx)
            out[:, :, m * ty:m * ty + vr, m * tx:m * tx + vc] = \
                Yt[:vr, :vc, :, :, ty, tx].transpose(3, 2, 0, 1)
    return out


def winograd_forward(d: np.ndarray, g: np.ndarray, m: int, pad: int,
                     U: np.ndarray | None = None) -> np.ndarray:
    """Whole-layer F(m x m, 3 x 3) forward (engine.py:198-254).

    d (N,C,H,W) and g (K,C,3,3) share a dtype (fp32 or fp64); output has the
    same dtype.  ``U`` may be a precomputed ``filter_transform`` (FX variant).
    """
    if d.dtype != g.dtype:
        raise ValueError("mixed precisions")
    N, C, H, W = d.shape
    K, C2, R, S = g.shape
    if C2 != C or R != 3 or S != 3:
        raise ValueError("shape mismatch")
    oh, ow = out_dims(H, W, R, S, pad)
    if U is None:
        U = filter_transform(g, m)
    V, th, tw = input_transform(d, m, pad, R)
    M = batched_matmul(U, V)
    return output_transform(M, m, K, N, th, tw, oh, ow, R)


# ---------------------------------------------------------------------------
# Direct-convolution oracle  (direct.py:82-114)
# ---------------------------------------------------------------------------
def direct_forward(d: np.ndarray, g: np.ndarray, pad: int,
                   accum=np.float64) -> np.ndarray:
    """Correlation with zero padding, reduction order c, v, u (direct.py:82-114)."""
    N, C, H, W = d.shape
    K, _, R, S = g.shape
    oh, ow = out_dims(H, W, R, S, pad)
    da = d.astype(accum, copy=False)
    ga = g.astype(accum, copy=False)
    y = np.zeros((N, K, oh, ow), dtype=accum)
    for c in range(C):
        for v in range(S):
            for u in range(R):
                ro, co = u - pad, v - pad
                xs, xe = max(0, -ro), min(oh, H - ro)
                ys, ye = max(0, -co), min(ow, W - co)
                if xs >= xe or ys >= ye:
                    continue
                win = da[:, c, xs + ro:xe + ro, ys + co:ye + co]
                y[:, :, xs:xe, ys:ye] += win[:, None] * ga[None, :, c, u, v, None, None]
    return y


def direct_grad_weights(d: np.ndarray, dy: np.ndarray, pad: int, R: int = 3, S: int = 3,
                        accum=np.float64) -> np.ndarray:
    """dG[k,c,u,v] = sum_i sum_{x,y} d[i,c,x+u-pad,y+v-pad] * dy[i,k,x,y]
    (direct.py:149-177): the fp64 ground truth of the weight gradient."""
    N, C, H, W = d.shape
    _, K, oh, ow = dy.shape
    da = d.astype(accum, copy=False)
    ya = dy.astype(accum, copy=False)
    dg = np.zeros((K, C, R, S), dtype=accum)
    for u in range(R):
        for v in range(S):
            ro, co = u - pad, v - pad
            xs, xe = max(0, -ro), min(oh, H - ro)
            ys, ye = max(0, -co), min(ow, W - co)
            if xs >= xe or ys >= ye:
                continue
            win = da[:, :, xs + ro:xe + ro, ys + co:ye + co]
            dg[:, :, u, v] = np.einsum("ichw,ikhw->kc", win, ya[:, :, xs:xe, ys:ye])
    return dg


def winograd_grad_weights(d: np.ndarray, dy: np.ndarray, pad: int) -> np.ndarray:
    """dL/dg via F(3x3, 2x2) (engine.py:278-328).

    dy is cut into non-overlapping 2x2 tiles (zero-filled past the output
    edge); each pairs with the 4x4 input patch at (2ty - pad, 2tx - pad).
    Uw = G dy_tile G^T (alpha^2, K, B), Vw = B^T d_tile B (alpha^2, B, C),
    M = Uw @ Vw per component (reduction over tiles B), dg = A^T M A.
    Arithmetic in the input dtype, as the reference.
    """
    if d.dtype != dy.dtype:
        raise ValueError("mixed precisions")
    N, C, H, W = d.shape
    _, K, oh, ow = dy.shape
    BT, G, AT = lowered(3, 2, d.dtype)
    mw, aw = 2, 4
    gh, gw = -(-oh // mw), -(-ow // mw)
    B = N * gh * gw
    yt = gather_tiles(dy, gh, gw, mw, mw, 0).reshape(B, K, mw, mw)
    dt = gather_tiles(d, gh, gw, mw, aw, pad).reshape(B, C, aw, aw)
    t = np.einsum("xr,bkrs->xbks", G, yt)
    Uw = np.ascontiguousarray(np.einsum("ys,xbks->xykb", G, t).reshape(aw * aw, K, B))
    t = np.einsum("xu,bcuv->xbcv", BT, dt)
    Vw = np.ascontiguousarray(np.einsum("yv,xbcv->xybc", BT, t).reshape(aw * aw, B, C))
    M = batched_matmul(Uw, Vw)
    M4 = M.reshape(aw, aw, K, C)
    t2 = np.einsum("mx,xykc->mykc", AT, M4)
    return np.ascontiguousarray(np.einsum("ny,mykc->kcmn", AT, t2))


def gflops_direct(N, C, H, W, K, pad, R=3, S=3, depth=1) -> float:
    """2*N*C*K*outH*outW*R*S / 1e9 * depth (direct.py:179-183)."""
    oh, ow = out_dims(H, W, R, S, pad)
    return 2.0 * N * C * K * oh * ow * R * S / 1e9 * depth


# VGG-E rows (label, C, H=W, K, depth), all pad=1 (suites.py:68-78)
VGG_E = (
    ("conv1.1", 3, 224, 64, 1),
    ("conv1.2", 64, 224, 64, 1),
    ("conv2.1", 64, 112, 128, 1),
    ("conv2.2", 128, 112, 128, 1),
    ("conv3.1", 128, 56, 256, 1),
    ("conv3.2", 256, 56, 256, 3),
    ("conv4.1", 256, 28, 512, 1),
    ("conv4.2", 512, 28, 512, 3),
    ("conv5", 512, 14, 512, 4),
)


def layer_inputs(N, C, H, W, K, seed: int, index: int, R: int = 3, S: int = 3):
    """Data seed seed+2i, filter seed seed+2i+1, U[-1,1) fp32 (commands.py:54-61)."""
    d = fill_uniform((N, C, H, W), seed + 2 * index)
    g = fill_uniform((K, C, R, S), seed + 2 * index + 1)
    return d, g
