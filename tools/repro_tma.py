import sys, torch
sys.path.insert(0, '/root/repo')
import paper_1509_09308_b200 as wb
cfg = wb.LayerConfig(N=1, C=64, H=20, W=20, K=64, pad=1)
for m in (2, 4):
    p = wb.WinogradPlan(cfg, m, "fp32")
    d = torch.rand((1, 64, 20, 20), device="cuda"); g = torch.rand((64, 64, 3, 3), device="cuda")
    y = p.forward(d, g=g); torch.cuda.synchronize(); print("ok", m, float(y.abs().sum()))
