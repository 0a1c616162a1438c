"""One non-FX forward of a single VGG-E layer (default conv5, F2 fp32, N=1),
for profiling the filter transform with ncu.

usage: python tools/filter_layer.py [C] [K] [H] [ALGO] [PREC] [BATCH]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else 512
K = int(sys.argv[2]) if len(sys.argv) > 2 else 512
H = int(sys.argv[3]) if len(sys.argv) > 3 else 14
algo = sys.argv[4] if len(sys.argv) > 4 else "f2x2"
prec = sys.argv[5] if len(sys.argv) > 5 else "fp32"
N = int(sys.argv[6]) if len(sys.argv) > 6 else 1
m, fx, _ = wb.parse_algo(algo)
cfg = wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
plan = wb.WinogradPlan(cfg, m, prec)
d = torch.rand((N, C, H, H), device="cuda") - 0.5
g = torch.rand((K, C, 3, 3), device="cuda") - 0.5
ws = plan.alloc_workspace()
y = torch.empty(plan.out_shape, device="cuda")
for _ in range(3):
    plan.forward(d, y=y, g=g, workspace=ws)
torch.cuda.synchronize()
print("ok")
