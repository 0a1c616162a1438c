"""Run one VGG-E layer forward a few times (for ncu captures).

usage: python tools/prof_layer.py LABEL M PREC BATCH [REPS] [BUDGET_MB] [FX]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402
from paper_1509_09308_b200.suites import VGG_E_ROWS  # noqa: E402

label, m, prec, batch = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
budget = int(sys.argv[6]) << 20 if len(sys.argv) > 6 else 0
fx = len(sys.argv) > 7 and sys.argv[7] == "fx"
row = [r for r in VGG_E_ROWS if r[0] == label][0]
_, C, H, K, _ = row
cfg = wb.LayerConfig(N=batch, C=C, H=H, W=H, K=K, pad=1)
plan = wb.WinogradPlan(cfg, m, prec, workspace_limit=budget)
d = torch.rand((batch, C, H, H), device="cuda") * 2 - 1
g = torch.rand((K, C, 3, 3), device="cuda") * 2 - 1
ws = plan.alloc_workspace()
y = torch.empty(plan.out_shape, device="cuda")
U = plan.filter_transform(g) if fx else None
for _ in range(reps):
    plan.forward(d, y=y, U=U, g=None if fx else g, workspace=ws)
torch.cuda.synchronize()
print(plan.info)
