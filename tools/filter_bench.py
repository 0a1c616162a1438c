"""Filter transform alone: device time per call (CUDA graph of 50 calls).
usage: python tools/filter_bench.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402

for (K, C, m, prec) in [(512, 512, 2, "fp32"), (512, 512, 4, "bf16"), (256, 256, 2, "fp32"),
                        (512, 256, 2, "fp32")]:
    plan = wb.WinogradPlan(wb.LayerConfig(N=1, C=C, H=14, W=14, K=K, pad=1), m, prec)
    g = torch.rand((K, C, 3, 3), device="cuda")
    U = plan.filter_transform(g)
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(50):
            plan.filter_transform(g, U=U, stream=torch.cuda.current_stream())
    for _ in range(3):
        gr.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        gr.replay()
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) / 250 * 1e3
    nb = K * C * 36 + plan.info["u_bytes"]
    print(f"K={K} C={C} F{m} {prec}: {us:.2f} us/call, {nb / us / 1e3:.0f} GB/s (in+out)")
