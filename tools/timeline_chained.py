"""Kernel timeline of one graph-replayed chained VGG-E forward (CUPTI).
usage: python tools/timeline_chained.py M PREC N"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1509_09308_b200.network import VGGEStack  # noqa: E402

m, prec, n = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
net = VGGEStack(n, m, prec, seed=0)
x = torch.rand(net.in_shape, device="cuda") * 2 - 1
out = torch.empty(net.out_shape, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    net.forward(x, out=out, stream=s)
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=s):
    net.forward(x, out=out, stream=torch.cuda.current_stream())
for _ in range(3):
    gr.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    gr.replay()
    torch.cuda.synchronize()
k = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
           if e.device_type.name == "CUDA")
t0 = k[0][0]
print(f"kernels {len(k)} span {k[-1][1] - t0:.1f} us")
for a, b, nm in k:
    print(f"{a - t0:8.1f} {b - t0:8.1f} {b - a:7.2f}  {nm[:70]}")
