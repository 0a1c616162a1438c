"""e2e arrangements of the default step (16 independent VGG-E layer calls, F2
fp32 N=1, host buffers): (a) bench.py's: wino_forward_host round-robin over 4
streams; (b) dedicated H2D and D2H streams (copies in call order) with each
call's kernels on its own stream, joined by events; (c) like (b) with two D2H
streams.  Diagnostic for the e2e leg (PCIe-bound).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402
from paper_1509_09308_b200.suites import VGG_E_ROWS  # noqa: E402

calls = []
for (lbl, C, H, K, depth) in VGG_E_ROWS:
    cfg = wb.LayerConfig(N=1, C=C, H=H, W=H, K=K, pad=1)
    plan = wb.WinogradPlan(cfg, 2, "fp32")
    for _ in range(depth):
        calls.append(dict(plan=plan,
                          dh=(torch.rand((1, C, H, H)) * 2 - 1).pin_memory(),
                          yh=torch.empty(plan.out_shape).pin_memory(),
                          d=torch.empty((1, C, H, H), device="cuda"),
                          y=torch.empty(plan.out_shape, device="cuda"),
                          g=torch.rand((K, C, 3, 3), device="cuda") * 2 - 1,
                          ws=plan.alloc_workspace(),
                          s=torch.cuda.Stream(), e_in=torch.cuda.Event(), e_out=torch.cuda.Event()))
gf = sum(2.0 * 1 * C * K * H * H * 9 / 1e9 * dep for (_, C, H, K, dep) in VGG_E_ROWS)
main = torch.cuda.current_stream()
rr = [torch.cuda.Stream() for _ in range(4)]
h2d, d2h, d2h2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def step_rr():
    for i, c in enumerate(calls):
        st = rr[i % 4]
        c["plan"].forward_host(c["dh"], c["yh"], c["d"], c["y"], g=c["g"], workspace=c["ws"],
                               stream=st)


def step_ded(nd2h):
    for i, c in enumerate(calls):
        with torch.cuda.stream(h2d):
            c["d"].copy_(c["dh"], non_blocking=True)
            c["e_in"].record(h2d)
        c["s"].wait_event(c["e_in"])
        c["plan"].forward(c["d"], y=c["y"], g=c["g"], workspace=c["ws"], stream=c["s"])
        c["e_out"].record(c["s"])
        ds = d2h if (nd2h == 1 or i % 2 == 0) else d2h2
        ds.wait_event(c["e_out"])
        with torch.cuda.stream(ds):
            c["yh"].copy_(c["y"], non_blocking=True)


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for st in rr + [h2d, d2h, d2h2] + [c["s"] for c in calls]:
        st.wait_event(a)
    for _ in range(reps):
        fn()
    for st in rr + [h2d, d2h, d2h2] + [c["s"] for c in calls]:
        ev = torch.cuda.Event()
        ev.record(st)
        main.wait_event(ev)
    b.record(main)
    b.synchronize()
    return a.elapsed_time(b) / reps


for name, fn in (("round-robin forward_host x4", step_rr), ("dedicated H2D/D2H streams", lambda: step_ded(1)),
                 ("dedicated H2D + 2 D2H streams", lambda: step_ded(2))):
    ms = timed(fn)
    print(f"{name:32s} {ms:.3f} ms/step  e2e {gf / ms:.1f} TFLOPS")
