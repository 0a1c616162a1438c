"""Kernel timeline of one VGG-E pass replayed from a CUDA graph (CUPTI via
torch.profiler): start/end of every kernel, so overlap and gaps are visible.
Diagnostic tool.

usage: python tools/timeline.py ALGO PREC BATCH [OUT.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402
from paper_1509_09308_b200.suites import VGG_E_ROWS  # noqa: E402

algo, prec, batch = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = sys.argv[4] if len(sys.argv) > 4 else None
m, fx, _ = wb.parse_algo(algo)
layers = []
rows = list(VGG_E_ROWS)
if os.environ.get("TL_ROTATE"):  # diagnostic: start the pass at another layer
    k = int(os.environ["TL_ROTATE"])
    rows = rows[k:] + rows[:k]
for (lbl, C, H, K, depth) in rows:
    cfg = wb.LayerConfig(N=batch, C=C, H=H, W=H, K=K, pad=1)
    plan = wb.WinogradPlan(cfg, m, prec)
    d = torch.rand((batch, C, H, H), device="cuda") * 2 - 1
    g = torch.rand((K, C, 3, 3), device="cuda") * 2 - 1
    layers.append((lbl, depth, plan, d, g, plan.alloc_workspace(),
                   torch.empty(plan.out_shape, device="cuda"),
                   plan.filter_transform(g) if fx else None))
s = torch.cuda.Stream()


def body():
    for (lbl, depth, plan, d, g, ws, y, U) in layers:
        for _ in range(depth):
            plan.forward(d, y=y, U=U, g=None if fx else g, workspace=ws,
                         stream=torch.cuda.current_stream())


with torch.cuda.stream(s):
    body()
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=s):
    body()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    gr.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        flush.fill_(1)
        gr.replay()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
kern = []
for e in evs:
    kern.append((e.time_range.start, e.time_range.end, e.name))
kern.sort()
# last replay: kernels after the last fill kernel
idx = max(i for i, k in enumerate(kern) if "fill" in k[2] or "elementwise" in k[2])
step = kern[idx + 1:]
t0 = step[0][0]
rows = [dict(start=k[0] - t0, end=k[1] - t0, dur=k[1] - k[0], name=k[2][:60]) for k in step]
print(f"kernels {len(rows)}  span {step[-1][1] - t0:.1f} us")
busy = 0.0
cur_s = cur_e = None
for r in rows:
    if cur_e is None or r["start"] > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = r["start"], r["end"]
    else:
        cur_e = max(cur_e, r["end"])
busy += cur_e - cur_s
print(f"busy (union of kernel intervals) {busy:.1f} us")
for r in rows:
    print(f"{r['start']:8.1f} {r['end']:8.1f} {r['dur']:7.2f}  {r['name']}")
if out:
    with open(out, "w") as fh:
        json.dump(rows, fh)
