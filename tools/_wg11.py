import sys, torch
sys.path.insert(0, '.')
import paper_1509_09308_b200 as wb
prec = sys.argv[1]
B, C, H, K = 8, 3, 224, 64
cfg = wb.LayerConfig(N=B, C=C, H=H, W=H, K=K, pad=1)
d = torch.rand((B, C, H, H), device="cuda") - 0.5
dy = torch.rand((B, K, H, H), device="cuda") - 0.5
ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(2):
    wb.grad_weights_device(d, dy, cfg, prec, workspace=ws, stream=torch.cuda.current_stream())
torch.cuda.synchronize()
