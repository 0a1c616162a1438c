"""Weight-gradient staging-chunk sweep: device time per VGG-E layer for several
Uw+Vw chunk budgets (WINO_WGRAD_CHUNK_MB; small chunks stay in L2).

usage: python tools/wgrad_chunk_sweep.py [BATCH] [PREC] [LAYER ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402
from paper_1509_09308_b200.suites import VGG_E_ROWS  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
only = set(sys.argv[3:])


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
    return a.elapsed_time(b) / reps * 1e3


ws = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
for (lbl, C, H, K, depth) in VGG_E_ROWS:
    if only and lbl not in only:
        continue
    cfg = wb.LayerConfig(N=B, C=C, H=H, W=H, K=K, pad=1)
    d = torch.rand((B, C, H, H), device="cuda") - 0.5
    dy = torch.rand((B, K, H, H), device="cuda") - 0.5
    row = []
    for mb in (0, 16, 24, 32, 48, 64, 96, 128):
        if mb:
            os.environ["WINO_WGRAD_CHUNK_MB"] = str(mb)
        else:
            os.environ.pop("WINO_WGRAD_CHUNK_MB", None)
        t = graph_time(lambda: wb.grad_weights_device(d, dy, cfg, prec, workspace=ws,
                                                      stream=torch.cuda.current_stream()))
        row.append(f"{mb or 'plan'}:{t:.1f}")
    os.environ.pop("WINO_WGRAD_CHUNK_MB", None)
    print(lbl, prec, " ".join(row), flush=True)
