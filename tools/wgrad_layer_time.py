"""Device time of one weight-gradient layer (conv1.1 shape by default; C as
argv[2]) by CUDA-graph replay; WINO_GEMM_DBG / WINO_NO_WGRAD_SMALLC apply.

usage: python tools/wgrad_layer_time.py PREC [C]
"""
import os, sys, torch
sys.path.insert(0, '.')
import paper_1509_09308_b200 as wb
prec = sys.argv[1]
B, C, H, K = 8, int(sys.argv[2]) if len(sys.argv) > 2 else 3, 224, 64
cfg = wb.LayerConfig(N=B, C=C, H=H, W=H, K=K, pad=1)
d = torch.rand((B, C, H, H), device="cuda") - 0.5
dy = torch.rand((B, K, H, H), device="cuda") - 0.5
ws = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
f = lambda: wb.grad_weights_device(d, dy, cfg, prec, workspace=ws, stream=torch.cuda.current_stream())
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    f()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    f()
g.replay(); g.replay()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    g.replay()
b.record(); b.synchronize()
print(prec, "C", C, "dbg", os.environ.get("WINO_GEMM_DBG", "0"), f"{a.elapsed_time(b) / 10 * 1e3:.1f} us")
