"""PCIe copy-bandwidth probe (pinned host <-> device): H2D alone, D2H alone and
both directions at once on two streams.  Diagnostic for the bench's e2e leg.

usage: python tools/pcie_probe.py [MB]
"""
import sys

import torch

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = mb << 18  # fp32 elements
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, device="cuda")
d_out = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


nb = n * 4
t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"{mb} MB: H2D {nb / t1 / 1e9:.1f} GB/s  D2H {nb / t2 / 1e9:.1f} GB/s  "
      f"both {2 * nb / t3 / 1e9:.1f} GB/s total ({t3 * 1e3:.2f} ms for {mb} MB each way)")
