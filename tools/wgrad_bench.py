"""Weight gradient (F(3x3,2x2), wino_grad_weights) per VGG-E layer: device time
(CUDA graph replay, warm) and effective TFLOPS = direct-conv-equivalent
2*N*C*K*H*W*9 / time, plus the forward of the same layer for comparison.

usage: python tools/wgrad_bench.py [BATCH] [PREC]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402
from paper_1509_09308_b200.suites import VGG_E_ROWS  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"


def graph_time(fn, reps=10):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    for _ in range(2):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps / 1e3


tot_w = tot_f = tot_gf = 0.0
print(f"{'layer':8s} {'wgrad us':>9s} {'TFLOPS':>7s} {'fwd F2 us':>9s}   (N={B}, {prec})")
for (lbl, C, H, K, depth) in VGG_E_ROWS:
    cfg = wb.LayerConfig(N=B, C=C, H=H, W=H, K=K, pad=1)
    d = torch.rand((B, C, H, H), device="cuda") - 0.5
    dy = torch.rand((B, K, H, H), device="cuda") - 0.5
    g = torch.rand((K, C, 3, 3), device="cuda") - 0.5
    ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    tw = graph_time(lambda: wb.grad_weights_device(d, dy, cfg, prec, workspace=ws,
                                                   stream=torch.cuda.current_stream()))
    plan = wb.WinogradPlan(cfg, 2, prec)
    wsf = plan.alloc_workspace()
    y = torch.empty(plan.out_shape, device="cuda")
    tf = graph_time(lambda: plan.forward(d, y=y, g=g, workspace=wsf,
                                         stream=torch.cuda.current_stream()))
    gf = 2.0 * B * C * K * H * H * 9 / 1e9
    print(f"{lbl:8s} {tw * 1e6:9.1f} {gf / tw / 1e3:7.1f} {tf * 1e6:9.1f}  x{depth}")
    tot_w += tw * depth
    tot_f += tf * depth
    tot_gf += gf * depth
print(f"{'TOTAL':8s} {tot_w * 1e6:9.1f} {tot_gf / tot_w / 1e3:7.1f} {tot_f * 1e6:9.1f}")
