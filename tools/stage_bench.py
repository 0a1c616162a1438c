"""Per-layer, per-stage device times of the VGG-E pass (CUDA events on the
launch stream, warm L2, no host gaps).  Diagnostic tool, not the bench.

usage: python tools/stage_bench.py ALGO PREC BATCH [REPS]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402
from paper_1509_09308_b200.suites import VGG_E_ROWS  # noqa: E402

algo, prec, batch = sys.argv[1], sys.argv[2], int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
budget = int(sys.argv[5]) << 20 if len(sys.argv) > 5 else 0
m, fx, _ = wb.parse_algo(algo)
s = torch.cuda.Stream()
tot = [0.0] * 5
print(f"{'layer':8s} {'bn':>3s} {'sp':>3s} {'ch':>3s} {'filter':>8s} {'input':>8s} {'gemm':>8s} "
      f"{'output':>8s} {'sum':>8s} {'plain':>8s} {'graph':>8s}  us/instance")
for (lbl, C, H, K, depth) in VGG_E_ROWS:
    cfg = wb.LayerConfig(N=batch, C=C, H=H, W=H, K=K, pad=1)
    plan = wb.WinogradPlan(cfg, m, prec, workspace_limit=budget)
    d = torch.rand((batch, C, H, H), device="cuda") * 2 - 1
    g = torch.rand((K, C, 3, 3), device="cuda") * 2 - 1
    ws = plan.alloc_workspace()
    y = torch.empty(plan.out_shape, device="cuda")
    U = plan.filter_transform(g) if fx else None
    kw = dict(U=U, g=None if fx else g, workspace=ws, stream=s)
    timer = wb.engine.StageTimer()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(s):
        for _ in range(3):
            plan.forward(d, y=y, **kw)
        for _ in range(reps):
            flush.fill_(1)  # host head start -> the timer sees device time only
            timer.gap()
            plan.forward_timed(d, y, timer, **kw)
    acc, _ = timer.read()
    acc = [a / reps * 1e3 for a in acc]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(reps):
            plan.forward(d, y=y, **kw)
        b.record(s)
    b.synchronize()
    plain = a.elapsed_time(b) / reps * 1e3
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        plan.forward(d, y=y, **kw)
    with torch.cuda.stream(s):
        gr.replay()
        a.record(s)
        for _ in range(reps):
            gr.replay()
        b.record(s)
    b.synchronize()
    graph = a.elapsed_time(b) / reps * 1e3
    i = plan.info
    print(f"{lbl:8s} {i['gemm_bn']:3d} {i['gemm_splits']:3d} {i['num_chunks']:3d} "
          + " ".join(f"{v:8.1f}" for v in acc) + f" {sum(acc):8.1f} {plain:8.1f} {graph:8.1f}"
          + f"  x{depth}")
    for j in range(4):
        tot[j] += acc[j] * depth
    tot[4] += graph * depth
print(f"{'TOTAL':8s} {'':3s} {'':3s} {'':3s} " + " ".join(f"{v:8.1f}" for v in tot[:4])
      + f" {sum(tot[:4]):8.1f} {'':8s} {tot[4]:8.1f}")
