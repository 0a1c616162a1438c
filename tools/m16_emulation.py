"""Emulation: F(4x4) with fp16 / bf16 operands (U, V), fp32 accumulation, and M staged in fp32
or bf16, against the fp64 direct convolution (round-2 decision: fp16 keeps fp32 M).
CPU only (torch fp64 einsums over the oracle's lowered matrices); diagnostic tool.
Measured: fp16 + fp32 M 0.73-0.78% max rel; fp16 + bf16 M 6.3-8.6%; bf16 + fp32 M 6.2-6.9%;
bf16 + bf16 M 8.7-9.6% (C/K = 256@28, 512@14, 64@56, N=1).
"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import winograd_oracle as O
def rnd(x, dt): return x.to(dt).to(torch.float64)
def wino(d, g, m, op_dt, m_dt):
    BT, G, AT = [torch.from_numpy(np.asarray(x, dtype=np.float64)) for x in O.lowered(m, 3, np.float32)]
    a = m + 2
    N, C, H, W = d.shape; K = g.shape[0]
    U = torch.einsum('ir,kcrs,js->ijkc', G, g, G)
    th, tw = (H + m - 1)//m, (W + m - 1)//m
    dp = torch.zeros(N, C, th*m + 2, tw*m + 2, dtype=torch.float64); dp[:, :, 1:H+1, 1:W+1] = d
    pt = dp.unfold(2, a, m).unfold(3, a, m)  # N C th tw a a
    V = torch.einsum('iu,nctyuv,jv->ijncty', BT, pt, BT)
    U, V = rnd(U, op_dt), rnd(V, op_dt)
    M = torch.einsum('ijkc,ijncty->ijnkty', U.float(), V.float()).double()  # fp32 accumulate
    M = rnd(M, m_dt) if m_dt is not None else M
    Y = torch.einsum('pi,ijnkty,qj->nktypq', AT, M, AT)
    return Y.permute(0,1,2,4,3,5).reshape(N, K, th*m, tw*m)[:, :, :H, :W]
for (N,C,H,K) in [(1,256,28,256),(1,512,14,512),(1,64,56,64)]:
    d = torch.from_numpy(O.fill_uniform((N,C,H,H), 3).astype(np.float64))
    g = torch.from_numpy(O.fill_uniform((K,C,3,3), 4).astype(np.float64))
    ref = torch.nn.functional.conv2d(d, g, padding=1)
    s = ref.abs().max().item()
    for op in (torch.float16, torch.bfloat16):
        for mdt in (None, torch.bfloat16):
            y = wino(d, g, 4, op, mdt)
            e = (y - ref).abs()
            print(f"C{C} H{H} F4 op={str(op)[6:]} M={'fp32' if mdt is None else 'bf16'}: max rel {e.max().item()/s:.3e} rms rel {(e.pow(2).mean().sqrt().item())/s:.3e}")
