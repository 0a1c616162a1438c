"""Launch-overhead calibration: per-kernel cost of a CUDA graph of tiny kernels
vs a graph of repeated small-layer forwards, under sustained load."""
import os
import subprocess
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402

clk = []
stop = threading.Event()


def sample():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        clk.append(out)
        stop.wait(0.05)


th = threading.Thread(target=sample, daemon=True)
th.start()
s = torch.cuda.Stream()
x = torch.zeros(1, device="cuda")


def timed_graph(fn, reps=20):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    with torch.cuda.stream(s):
        for _ in range(3):
            g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            g.replay()
        b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


t = timed_graph(lambda: [x.add_(1) for _ in range(200)])
print(f"torch tiny kernel in graph: {t / 200:.2f} us/kernel")
for (C, H, K, m, prec, N) in [(16, 8, 16, 2, "fp32", 1), (16, 8, 16, 4, "bf16", 1), (512, 14, 512, 4, "bf16", 1), (512, 14, 512, 2, "fp32", 1),
                              (64, 56, 64, 2, "fp32", 1), (256, 56, 256, 4, "bf16", 1)]:
    cfg = wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
    plan = wb.WinogradPlan(cfg, m, prec)
    d = torch.rand((N, C, H, H), device="cuda")
    g = torch.rand((K, C, 3, 3), device="cuda")
    ws = plan.alloc_workspace()
    y = torch.empty(plan.out_shape, device="cuda")
    U = plan.filter_transform(g)
    torch.cuda.synchronize()
    for label, kw in (("fx", dict(U=U)), ("non-fx", dict(g=g))):
        reps = 50
        tt = timed_graph(lambda: [plan.forward(d, y=y, workspace=ws, stream=torch.cuda.current_stream(), **kw)
                                  for _ in range(reps)])
        print(f"C={C} H={H} K={K} F{m} {prec} N={N} {label}: {tt / reps:.1f} us/layer "
              f"({plan.info['launches_per_forward'] + (1 if label == 'non-fx' else 0)} kernels)")
stop.set()
th.join()
vals = [int(v) for v in clk if v.isdigit()]
print("sm clocks MHz: min", min(vals), "median", sorted(vals)[len(vals) // 2], "max", max(vals),
      "n", len(vals))
