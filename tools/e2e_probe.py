"""Copy-only model of the bench's e2e leg: the VGG-E layer calls' H2D input and
D2H output copies (pinned host memory), round-robin over S streams, for a few
call orders.  Tells how close the e2e number is to the PCIe bound.

usage: python tools/e2e_probe.py [BATCH]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1509_09308_b200.suites import VGG_E_ROWS  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
calls = []
for (lbl, C, H, K, depth) in VGG_E_ROWS:
    for _ in range(depth):
        calls.append((lbl, B * C * H * H, B * K * H * H))


def run(order, S, steps=5):
    streams = [torch.cuda.Stream() for _ in range(S)]
    bufs = [[(torch.empty(i, pin_memory=True), torch.empty(i, device="cuda"),
              torch.empty(o, device="cuda"), torch.empty(o, pin_memory=True))
             for (_, i, o) in calls] for _ in range(S)]

    def step():
        for n, ci in enumerate(order):
            si = n % S
            hi, di, do, ho = bufs[si][ci]
            with torch.cuda.stream(streams[si]):
                di.copy_(hi, non_blocking=True)
                ho.copy_(do, non_blocking=True)

    step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    for s in streams:
        s.wait_stream(cur)
    for _ in range(steps):
        step()
    for s in streams:
        cur.wait_stream(s)
    b.record(cur)
    b.synchronize()
    return a.elapsed_time(b) / steps


def run_split(steps=5):
    """All H2D copies on one stream, all D2H copies on another; D2H of call i
    waits for H2D of call i (stands in for the compute dependency)."""
    hs, ds = torch.cuda.Stream(), torch.cuda.Stream()
    bufs = [(torch.empty(i, pin_memory=True), torch.empty(i, device="cuda"),
             torch.empty(o, device="cuda"), torch.empty(o, pin_memory=True))
            for (_, i, o) in calls]

    def step():
        for hi, di, do, ho in bufs:
            with torch.cuda.stream(hs):
                di.copy_(hi, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(hs)
            ds.wait_event(ev)
            with torch.cuda.stream(ds):
                ho.copy_(do, non_blocking=True)

    step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    hs.wait_stream(cur)
    ds.wait_stream(cur)
    for _ in range(steps):
        step()
    cur.wait_stream(hs)
    cur.wait_stream(ds)
    b.record(cur)
    b.synchronize()
    return a.elapsed_time(b) / steps


nb_in = sum(i for _, i, _ in calls) * 4
nb_out = sum(o for _, _, o in calls) * 4
print(f"batch {B}: H2D {nb_in / 1e6:.1f} MB, D2H {nb_out / 1e6:.1f} MB per step")
n = len(calls)
orders = {"network": list(range(n)), "reversed": list(range(n))[::-1],
          "interleaved": [x for pair in zip(range(n // 2), range(n - 1, n // 2 - 1, -1)) for x in pair]}
for name, order in orders.items():
    for S in (2, 4, 8):
        ms = run(order, S)
        print(f"{name:12s} S={S}: {ms:.3f} ms/step  ({(nb_in + nb_out) / ms / 1e6:.1f} GB/s)")
ms = run_split()
print(f"split h2d/d2h streams: {ms:.3f} ms/step  ({(nb_in + nb_out) / ms / 1e6:.1f} GB/s)")
