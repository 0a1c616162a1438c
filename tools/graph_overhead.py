"""Graph-launch overhead probe: device time of a replayed graph holding one tiny
kernel, one VGG-E pass, and two passes, each step bracketed by CUDA events after
a 256 MB L2 flush (the bench's arrangement).  Diagnostic.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402
from paper_1509_09308_b200.suites import VGG_E_ROWS  # noqa: E402

s = torch.cuda.Stream()
layers = []
for (lbl, C, H, K, depth) in VGG_E_ROWS:
    cfg = wb.LayerConfig(N=1, C=C, H=H, W=H, K=K, pad=1)
    plan = wb.WinogradPlan(cfg, 2, "fp32")
    for _ in range(depth):
        d = torch.rand((1, C, H, H), device="cuda") * 2 - 1
        g = torch.rand((K, C, 3, 3), device="cuda") * 2 - 1
        layers.append((plan, d, g, plan.alloc_workspace(), torch.empty(plan.out_shape, device="cuda")))
tiny = torch.zeros(1, device="cuda")


def one_pass():
    for (plan, d, g, ws, y) in layers:
        plan.forward(d, y=y, g=g, workspace=ws, stream=torch.cuda.current_stream())


def capture(fn):
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        fn()
    return gr


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
graphs = {"tiny kernel": capture(lambda: tiny.add_(1)), "1 pass": capture(one_pass),
          "2 passes": capture(lambda: (one_pass(), one_pass()))}
for name, gr in graphs.items():
    for _ in range(5):
        gr.replay()
    torch.cuda.synchronize()
    ts = []
    for flushed in (True, False):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
        with torch.cuda.stream(s):
            for a, b in evs:
                if flushed:
                    flush.fill_(1)
                a.record(s)
                gr.replay()
                b.record(s)
        torch.cuda.synchronize()
        ts.append(sorted(a.elapsed_time(b) * 1e3 for a, b in evs)[15])
    print(f"{name:12s} median us: flushed {ts[0]:8.1f}   back-to-back {ts[1]:8.1f}")
