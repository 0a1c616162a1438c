"""Run one layer's forward REPS times (profiling driver for ncu).

usage: python tools/one_layer.py C H K N m prec [reps] [fx]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402

C, H, K, N, m = (int(x) for x in sys.argv[1:6])
prec = sys.argv[6]
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
fx = len(sys.argv) > 8 and sys.argv[8] == "fx"
cfg = wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
plan = wb.WinogradPlan(cfg, m, prec)
d = torch.rand((N, C, H, H), device="cuda") * 2 - 1
g = torch.rand((K, C, 3, 3), device="cuda") * 2 - 1
ws = plan.alloc_workspace()
y = torch.empty(plan.out_shape, device="cuda")
U = plan.filter_transform(g) if fx else None
for _ in range(reps):
    plan.forward(d, y=y, U=U, g=None if fx else g, workspace=ws)
torch.cuda.synchronize()
print(plan.info)
